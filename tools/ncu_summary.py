#!/usr/bin/env python
"""Summarise ncu launch lists and full captures into the tables committed under profiles/.

    python tools/ncu_summary.py launches <launches.csv>      # per-kernel time and share of the step
    python tools/ncu_summary.py metrics <capture.ncu-rep>    # key roofline metrics per captured launch
    python tools/ncu_summary.py traffic <capture.ncu-rep> N  # DRAM bytes of the CN launches per iteration
    python tools/ncu_summary.py stalls <capture.ncu-rep>     # stall reasons + hottest SASS lines
"""
import csv
import io
import re
import subprocess
import sys
from collections import OrderedDict


def _short(name: str) -> str:
    name = re.sub(r"\(metldpc::CodeDev.*$|\(CodeDev.*$", "", name)
    name = name.replace("metldpc::", "").replace("void ", "")
    return name.strip()


def launches(path: str) -> str:
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = OrderedDict()
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
        k = _short(r[ik])
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + v)
    tot = sum(t for _, t in agg.values())
    out = io.StringIO()
    out.write(f"{'launches':>8} {'total us':>12} {'mean us':>10} {'share':>7}  kernel\n")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.write(f"{n:8d} {t:12.1f} {t / n:10.1f} {100 * t / tot:6.1f}%  {k}\n")
    out.write(f"{'':8s} {tot:12.1f} us total (ncu-serialised, cold-cache per launch)\n")
    return out.getvalue()


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second"]


def metrics(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = io.StringIO()
    for r in rows[2:]:
        out.write(_short(r[hdr.index("Kernel Name")]) + "\n")
        for k in KEYS:
            if k in hdr:
                out.write(f"    {k:62s} {r[hdr.index(k)]:>16s} {units[hdr.index(k)]}\n")
        rb = float(r[hdr.index("dram__bytes_read.sum")]) * (1e9 if units[hdr.index("dram__bytes_read.sum")] == "Gbyte" else 1e6 if units[hdr.index("dram__bytes_read.sum")] == "Mbyte" else 1)
        wb = float(r[hdr.index("dram__bytes_write.sum")]) * (1e9 if units[hdr.index("dram__bytes_write.sum")] == "Gbyte" else 1e6 if units[hdr.index("dram__bytes_write.sum")] == "Mbyte" else 1)
        out.write(f"    {'dram bytes (read + write)':62s} {rb + wb:16.0f} byte\n")
    return out.getvalue()


def _bytes(v: str, unit: str) -> float:
    return float(v.replace(",", "")) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(unit, 1.0)


def traffic(path: str, iterations: int) -> str:
    """DRAM bytes (read + write) of the captured CN launches per iteration, as the JSON
    bench.py reads for roofline.traffic (profiles/cn_traffic.json)."""
    import json
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    ik = hdr.index("Kernel Name")
    tot, kernels = 0.0, []
    for r in rows[2:]:
        b = _bytes(r[ir], units[ir]) + _bytes(r[iw], units[iw])
        tot += b
        kernels.append({"kernel": _short(r[ik]), "dram_bytes": b})
    return json.dumps({"source": path, "iterations": iterations, "dram_bytes_per_launch": tot / iterations,
                       "note": "sum over the CN-phase launches of one iteration (all degree classes), one 64-lane group",
                       "launches": kernels}, indent=1) + "\n"


def stalls(path: str, top: int = 12) -> str:
    """Warp-stall reasons per issued instruction and the hottest SASS lines of each captured kernel."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    out = io.StringIO()
    for r in rows[2:]:
        out.write(_short(r[hdr.index("Kernel Name")]) + "  (warps stalled per issued instruction)\n")
        st = []
        for i, h in enumerate(hdr):
            m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", h)
            if m:
                try:
                    st.append((float(r[i]), m.group(1)))
                except ValueError:
                    pass
        for v, name in sorted(st, reverse=True)[:8]:
            out.write(f"    {name:28s} {v:8.3f}\n")
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    i = 0
    while i < len(rows):
        if rows[i] and rows[i][0] == "Kernel Name":
            name = _short(rows[i][1])
            hdr = rows[i + 1]
            body = []
            i += 2
            while i < len(rows) and len(rows[i]) == len(hdr):
                body.append(dict(zip(hdr, rows[i])))
                i += 1
            def f(x):
                try:
                    return float(x)
                except ValueError:
                    return 0.0
            tot = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in body) or 1.0
            out.write(f"{name}: hottest SASS lines (share of stall samples)\n")
            for d in sorted(body, key=lambda d: -f(d["Warp Stall Sampling (All Samples)"]))[:top]:
                out.write(f"    {100 * f(d['Warp Stall Sampling (All Samples)']) / tot:5.1f}%  {d['Source'].strip()[:70]}\n")
        else:
            i += 1
    return out.getvalue()


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "stalls":
        sys.stdout.write(stalls(path))
    elif mode == "traffic":
        sys.stdout.write(traffic(path, int(sys.argv[3]) if len(sys.argv) > 3 else 1))
    else:
        sys.stdout.write(launches(path) if mode == "launches" else metrics(path))
