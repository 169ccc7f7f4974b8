#!/usr/bin/env python
"""bench.py -- throughput of the batched syndrome BP decoder (arXiv 1711.01783 hot path).

Workload (BASELINE.json configs[2], "C3"): a rate-0.1 MET-LDPC stand-in code with every Table-1
count of the paper's (n = 10^6; default the density-evolution-optimised r0.1de, R29),
SNR 0.161, N = 100 iterations with per-frame syndrome early termination and lane refill.  Input
(--input): the channel LLRs of the virtual BIAWGN channel MD reconciliation creates (default)
or the 8-D MD reconciliation output itself (--input md: metldpc_llr_from_md inside the step).  One
step = one pass of the whole hot path over one batch resident in HBM: [LLRs from MD output ->]
decode (metldpc_decode) -> FER counters (metldpc_batch_counters, NCCL all-reduce when N > 1).
Frames shard across ranks (frame f -> rank f mod G, weak scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.  `value` = decoded Mb/s (n bits per frame, the paper's
Table-1 convention) over all ranks, device-timed with CUDA events
(max over ranks); `e2e` = the same through metldpc_decode_host / metldpc_decode_md_host from
pinned host buffers (H2D + D2H inside the timed region); `roofline` = the check-node update phase
(dominant kernel) against the measured HBM copy bandwidth; `cpu_baseline` = the CPU
oracle (oracle/, fp32 replay M3) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decoded info Mb/s (rate-0.1 n=1e6) at 1/2/4/8 B200; HBM GB/s vs peak"
PAPER_MBPS = 30.39           # PAPER.md Table 1 (lines 69-72), rate 0.1, TITAN Xp, 64 codewords
# Table 1 "Speed" row per rate (BASELINE.md lines 31-37): (skip, no skip)
PAPER_TABLE1_MBPS = {"r0.1": (30.39, 27.54), "r0.05": (21.23, 18.49), "r0.02": (16.41, 14.00)}


# stand-in family -> the Table-1 column (code rate) it reproduces the counts of
RATE_COLUMN = {"r0.1": "r0.1", "r0.1de": "r0.1", "r0.05": "r0.05", "r0.02": "r0.02"}


def paper_mbps(a) -> float | None:
    if a.n != 1_000_000 or a.family not in RATE_COLUMN:
        return None
    return PAPER_TABLE1_MBPS[RATE_COLUMN[a.family]][1 if a.no_skip else 0]


def vs_baseline(a, value: float) -> float | None:
    """value / the paper's Table-1 speed only for the paper's own flow (fixed N, no early
    termination): BASELINE.md's numbers are for that workload; with early termination the
    workload differs and the paper's number is context only (baseline_context)."""
    p = paper_mbps(a)
    return (value / p) if (p and a.no_et) else None
SUSTAINED_NOTE = "HBM peak = MEASURED_PEAKS.json hbm_gbs (STREAM-style copy, measured)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--family", default="r0.1de",
                    help="stand-in code: r0.1de (DE-optimised, default), r0.1 (round-1 stand-in), r0.05, r0.02")
    ap.add_argument("--input", choices=["biawgn", "md"], default="biawgn",
                    help="biawgn: channel LLRs of the virtual BIAWGN channel at --snr (P:20, DESIGN.md R31); "
                         "md: 8-D MD reconciliation output through metldpc_llr_from_md (R13)")
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--snr", type=float, default=0.161)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--frames", type=int, default=4096,
                    help="frames per GPU per step (a streaming decode's fill and drain, about one frame's "
                         "decoding time, is amortised over the batch)")
    ap.add_argument("--distinct", type=int, default=64, help="distinct frames generated per rank (tiled)")
    ap.add_argument("--rule", choices=["exact", "lut"], default="exact")
    ap.add_argument("--no-et", action="store_true")
    ap.add_argument("--no-refill", action="store_true",
                    help="group mode instead of lane refill (metldpc_config_t.lane_refill = 0)")
    ap.add_argument("--no-skip", action="store_true",
                    help="iterate degree-1 VNs too (Table 1 'without skipping', METLDPC_CODE_NO_SKIP)")
    ap.add_argument("--lanes", type=int, default=64)
    ap.add_argument("--msg-bits", type=int, choices=[32, 16], default=32,
                    help="edge-message storage: fp32 or 16-bit rint(2^10 r) (DESIGN.md R28/N7)")
    ap.add_argument("--groups", type=int, default=1, help="lane groups decoded concurrently per GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--data-key", type=int, default=0)
    return ap.parse_args()


# ----------------------------------------------------------------------------- inputs

def _gen_one(args):
    family, n, snr, key, fid, kind = args
    from synth.codes import make_met_code
    from synth.frames import gen_frame, gen_frame_biawgn
    code = make_met_code(family, n)
    if kind == "biawgn":
        f = gen_frame_biawgn(code, snr, key, fid)
        return f["llr"], None, f["synd"]
    f = gen_frame(code, snr, key, fid)
    return f["v"], f["xnorm"], f["synd"]


def gen_frames(a, frame_ids):
    """(v, xnorm, S_B) per frame for --input md; (lambda, None, S_B) for --input biawgn."""
    from multiprocessing import get_context
    jobs = [(a.family, a.n, a.snr, a.data_key, int(f), a.input) for f in frame_ids]
    procs = max(1, min(len(jobs), (os.cpu_count() or 4) // 2, 32))
    with get_context("fork").Pool(procs) as pool:
        out = pool.map(_gen_one, jobs)
    xn = None if a.input == "biawgn" else np.stack([o[1] for o in out])
    return (np.stack([o[0] for o in out]), xn, np.stack([o[2] for o in out]))


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ----------------------------------------------------------------------------- CPU oracle (baseline / reference)

def oracle_throughput(a, code, v, xn, synd, budget_s: float, threads: int | None = None) -> dict:
    """The oracle M3 (fp32 replay, as it stands) decoding frames on host threads, one frame
    per thread.  Bounded sample: T frames x I iterations (I <= N) so it costs ~budget_s;
    throughput is normalised to the workload's N iterations per frame."""
    from oracle import bp
    T = threads or max(1, min(host_cores(), 32, len(v)))
    lam = [(bp.llr_from_md_f32(v[i % len(v)], xn[i % len(v)], a.snr) if xn is not None else v[i % len(v)])
           for i in range(T)]
    t0 = time.perf_counter()
    bp.decode(code, lam[0], synd[0], 1, early_term=not a.no_et, rule=_rule(a), prec=32, no_skip=a.no_skip,
              msg16=a.msg_bits == 16)
    t_iter = max(time.perf_counter() - t0, 1e-3)
    I = int(max(1, min(a.iters, budget_s / t_iter)))

    def one(i):
        return bp.decode(code, lam[i], synd[i % len(synd)], I, early_term=not a.no_et, rule=_rule(a), prec=32,
                         no_skip=a.no_skip, msg16=a.msg_bits == 16)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(T) as ex:
        res = list(ex.map(one, range(T)))
    dt = time.perf_counter() - t0
    iters_done = sum(r["iters"] for r in res)
    bits = T * code.n * (iters_done / T) / a.iters        # frames-equivalent at N iterations
    return {"value": bits / dt / 1e6, "unit": "Mb/s", "cores": T, "kind": "oracle",
            "sample": f"{T} frames (one per host thread) x {I} of N={a.iters} iterations, oracle M3 (fp32 replay, "
                      f"oracle/bp_oracle.c) on n={code.n}; throughput normalised to N iterations/frame; "
                      f"{dt:.1f} s wall"}


def _rule(a):
    return 0 if a.rule == "exact" else 1


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = [r.split(",") for r in Path(self.f.name).read_text().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows if len(r) >= 9 for k in range(4) if r[5 + k].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- main

def measured_peak_gbs() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def workload_name(a) -> str:
    tag = {"r0.1": "C3", "r0.1de": "C3", "r0.05": "C4", "r0.02": "C6"}.get(a.family, "custom") if a.n == 1_000_000 else "custom"
    return (f"{tag}: MET-LDPC {a.family} stand-in n={a.n}, SNR {a.snr}, max {a.iters} iterations "
            f"{'fixed' if a.no_et else 'with per-frame syndrome early termination'}, "
            f"{a.frames} frames/GPU per step"
            f"{', degree-1 VNs iterated (no skip)' if a.no_skip else ''}"
            f"{', 16-bit edge messages' if a.msg_bits == 16 else ''}, "
            + ("BIAWGN channel LLR input (the virtual channel of MD reconciliation, P:20)" if a.input == "biawgn"
               else "8-D MD LLR input"))


def run_reference(a, rank: int, world: int):
    if rank != 0:
        return
    from synth.codes import make_met_code
    code = make_met_code(a.family, a.n)
    v, xn, synd = gen_frames(a, range(min(a.distinct, 32)))
    T = max(1, min(host_cores(), 32))
    budget = max(2.0, 150.0 / max(1, a.steps + a.warmup))
    for _ in range(a.warmup):
        oracle_throughput(a, code, v, xn, synd, budget, T)
    vals, walls = [], []
    last = None
    for _ in range(a.steps):
        t0 = time.perf_counter()
        last = oracle_throughput(a, code, v, xn, synd, budget, T)
        walls.append(time.perf_counter() - t0)
        vals.append(last["value"])
    value = statistics.mean(vals)
    cpu = dict(last)
    cpu["value"] = value
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "Mb/s", "n_gpus": a.gpus,
           "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * statistics.mean(walls),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": vs_baseline(a, value), "dtype": "f32",
           "data": "synthetic", "config": {"workload": workload_name(a), "rule": a.rule.upper()},
           "cpu_baseline": cpu,
           "e2e": {"value": value, "unit": "Mb/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "gpu_launches": 0}
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------------- rank logic (shared with tests)

def spawn_ranks(a) -> int | None:
    """`python bench.py --gpus N` without a torchrun environment: launch N ranks (one per GPU)
    through torch.distributed.run on 127.0.0.1 and return its exit code; None if this process
    is already a rank (or N = 1)."""
    if a.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def rank_frame_ids(n_distinct: int, rank: int, world: int):
    """Global frame ids of this rank: f with f mod world == rank."""
    from paper_1711_01783_b200 import dist as D
    return D.shard_frames(range(n_distinct * world), rank, world)


def timed_steps(step, steps: int, warmup: int, sync, barrier, timer, on_start=None) -> float:
    """W untimed warm-up steps, then EXACTLY K timed steps bracketed by barrier + sync on
    both sides; step(i) gets the timed step's index (None during warm-up); on_start runs
    between the warm-up and the timed region.  Returns this rank's time in ms from `timer`
    (CUDA events on the launch stream in bench)."""
    for _ in range(max(warmup, 0)):
        step(None)
    sync()
    if on_start is not None:
        on_start()
        sync()
    barrier()
    t = timer
    t.start()
    for i in range(steps):
        step(i)
    t.stop()
    sync()
    barrier()
    return t.ms()


def gather_frames(iters, conv, world: int):
    """All-gather of the per-frame (iterations, converged) of the last step:
    returns int64 [world * F] arrays in global frame order (rank r's local frame i is
    global frame i * world + r, the f mod world sharding)."""
    import torch
    import torch.distributed as dist
    pair = torch.stack([iters.to(torch.int32), conv.to(torch.int32)]).contiguous()   # [2, F]
    if world > 1:
        parts = [torch.empty_like(pair) for _ in range(world)]
        dist.all_gather(parts, pair)
        out = torch.stack(parts)
    else:
        out = pair[None]
    out = out.cpu().numpy()                                                     # [world, 2, F]
    glob = out.transpose(1, 2, 0).reshape(2, -1)                                # frame i*world + r
    return glob[0].astype(np.int64), glob[1].astype(np.int64)


def summarize_counts(total, it_glob, cv_glob, frames_per_step: int) -> dict:
    """Counters summed over ranks and timed steps (k_counters + all-reduce), plus the
    per-frame picture of the last step from the all-gather."""
    frames_c, conv_c, iters_c, bad_c = (int(x) for x in total)
    valid = it_glob >= 0
    hist = np.bincount(it_glob[valid], minlength=1)
    return {"frames_timed": frames_c, "converged_timed": conv_c, "invalid_timed": bad_c,
            "fer": 1.0 - conv_c / max(1, frames_c), "mean_iters": iters_c / max(1, frames_c - bad_c),
            "last_step_frames": int(it_glob.size), "last_step_converged": int(cv_glob.sum()),
            "last_step_iters_hist": {str(k): int(v) for k, v in enumerate(hist) if v},
            "frames_per_step": frames_per_step}


# ----------------------------------------------------------------------------- main

def main():
    a = parse()
    rc = spawn_ranks(a) if a.impl == "ours" else None   # the reference arm is rank 0 alone
    if rc is not None:
        sys.exit(rc)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != a.gpus and "WORLD_SIZE" in os.environ:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}")
    if a.impl == "reference":
        return run_reference(a, rank, world)

    import torch
    import torch.distributed as dist
    from paper_1711_01783_b200 import binding as B
    from paper_1711_01783_b200 import dist as D
    from paper_1711_01783_b200 import metrics
    from paper_1711_01783_b200.build import build
    from synth.codes import make_met_code

    if rank == 0:
        build()
    torch.cuda.set_device(local)
    if world > 1:
        # the communicator's init lines (nranks, NVLS) go to stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist.barrier()
        if rank != 0:
            build()
        assert dist.get_world_size() == a.gpus
    dev = torch.device("cuda", local)
    code = make_met_code(a.family, a.n)
    st = code.stats()
    F = a.frames
    # frames of this rank: global ids f with f mod world == rank; ND distinct ones tiled to F
    ND = min(a.distinct, F)
    ids = rank_frame_ids(ND, rank, world)
    v_np, xn_np, sy_np = gen_frames(a, ids)       # biawgn: v_np holds the LLRs, xn_np is None
    rep = (F + ND - 1) // ND
    v = torch.from_numpy(np.tile(v_np, (rep, 1))[:F]).to(dev)
    xn = torch.from_numpy(np.tile(xn_np, (rep, 1))[:F]).to(dev) if xn_np is not None else None
    sy = torch.from_numpy(np.tile(sy_np, (rep, 1))[:F].view(np.int32)).to(dev)

    hc = B.Code(code, device=local, no_skip=a.no_skip)
    st = dict(st, iter_edges=hc.info.iter_edges, n_deg1=hc.info.n_deg1, n_active=hc.info.n_active)
    dec = B.Decoder(hc, F, rule=_rule(a), max_iter=a.iters, early_term=not a.no_et, lanes_per_group=a.lanes,
                    groups_in_flight=a.groups, lane_refill=not a.no_refill, msg_bits=a.msg_bits)
    llr = torch.empty_like(v)
    nw = (a.n + 31) // 32
    bits = torch.empty((F, nw), dtype=torch.int32, device=dev)
    iters = torch.empty(F, dtype=torch.int32, device=dev)
    conv = torch.empty(F, dtype=torch.uint8, device=dev)
    # one counter row per timed step (metldpc_batch_counters adds into its row; the row is
    # then all-reduced over the ranks -- the step's only exchange); warm-up uses a scratch row
    cnt = torch.zeros((a.steps + 1, 4), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream()

    def step(i):
        row = cnt[a.steps if i is None else i]
        if a.input == "md":
            dec.llr_from_md(v, xn, a.snr, out=llr)
            dec.decode(llr, sy, out=(bits, iters, conv))
        else:
            dec.decode(v, sy, out=(bits, iters, conv))
        dec.counters(iters, conv, row)
        D.reduce_counters(row)          # NCCL all-reduce when world > 1

    class CudaTimer:
        def start(self):
            self.e0 = torch.cuda.Event(enable_timing=True)
            self.e1 = torch.cuda.Event(enable_timing=True)
            self.e0.record(stream)

        def stop(self):
            self.e1.record(stream)

        def ms(self):
            return self.e0.elapsed_time(self.e1)

    def barrier():
        if world > 1:
            dist.barrier()

    dec.set_profiling(False)              # the timed region runs the production path (graph loop)
    holder = {}

    def on_start():                       # after warm-up: zero the launch count, start the clock sampler
        dec.reset_profile()
        holder["s"] = ClockSampler(local) if local == 0 or world == 1 else None

    ms_rank = timed_steps(step, a.steps, a.warmup, torch.cuda.synchronize, barrier, CudaTimer(), on_start)
    sampler = holder.get("s")
    clocks = sampler.stop() if sampler else None
    prof = dec.profile()
    ms_max = D.max_over_ranks(ms_rank, device=dev)
    total = cnt[:a.steps].sum(0).cpu().numpy()           # already summed over ranks per step
    it_glob, cv_glob = gather_frames(iters, conv, world)
    counts = summarize_counts(total, it_glob, cv_glob, F * world)
    frames_total = F * world * a.steps
    value = frames_total * a.n / (ms_max / 1e3) / 1e6

    # ---- roofline of the dominant kernel (check-node update phase), live CUDA-event timing.
    # Per-kernel events need the host-enqueued loop (the graph loop has no per-launch events)
    # and kernels of different groups must not overlap, so the kernel durations come from an
    # isolated pass: one 64-lane group in flight, same data, same process.
    # fixed N (no early termination): every launch does a whole pass over the 64 lanes, so the
    # per-launch time is the kernel's, not an average with early-exited launches
    iso = B.Decoder(hc, min(F, a.lanes), rule=_rule(a), max_iter=a.iters, early_term=False,
                    lanes_per_group=a.lanes, groups_in_flight=1, msg_bits=a.msg_bits)
    Fi = min(F, a.lanes)
    outi = (bits[:Fi], iters[:Fi], conv[:Fi])
    lam_dev = llr if a.input == "md" else v            # the step's LLRs (md: converted by the last step)
    iso.decode(lam_dev[:Fi], sy[:Fi], out=outi)
    torch.cuda.synchronize()
    iso.reset_profile()
    iso.set_profiling(True)
    for _ in range(2):
        iso.decode(lam_dev[:Fi], sy[:Fi], out=outi)
    torch.cuda.synchronize()
    prof_k = iso.profile()
    iso.close()
    kernel_timing = ("isolated pass: one 64-lane group in flight, fixed N (every launch a full pass), CUDA events "
                     "on the launch stream")
    bm = metrics.bytes_per_cw_iter(st["iter_edges"], st["n_deg1"], st["n_active"], st["m"], s_r=a.msg_bits // 8)
    peak, peak_src = measured_peak_gbs()
    cn_gbs = prof_k["cn_lane_iters"] * bm["cn"] / (prof_k["cn_ms"] / 1e3) / 1e9 if prof_k["cn_ms"] > 0 else None
    # ncu DRAM bytes of the CN phase, captured for one workload (profiles/cn_traffic.json):
    # reported only on a line of that workload
    traffic = traffic_prod = None
    tpath = ROOT / "profiles" / "cn_traffic.json"
    if tpath.exists():
        try:
            tj_all = json.loads(tpath.read_text())
            for tj in (tj_all if isinstance(tj_all, list) else [tj_all]):
                w = tj.get("workload", {})
                if (w.get("family"), w.get("n"), w.get("no_skip", False), w.get("lanes", 64),
                        str(w.get("rule", "exact")).lower(), w.get("msg_bits", 32)) != \
                        (a.family, a.n, bool(a.no_skip), a.lanes, a.rule, a.msg_bits):
                    continue
                traffic = tj.get("dram_bytes_per_launch")
                pg = tj.get("production_graph", {})
                traffic_prod = pg.get("dram_bytes_per_pass")
                if traffic_prod and pg.get("graph_ms_per_pass"):
                    # SURVEY 8(d)'s second fraction: ncu-measured DRAM bytes / time of a whole
                    # production pass (same capture), against the same peak
                    traffic_prod = {"bytes": traffic_prod, "ms": pg["graph_ms_per_pass"],
                                    "dram_gbs": traffic_prod / pg["graph_ms_per_pass"] / 1e6}
                break
        except Exception:
            traffic = traffic_prod = None
    # codeword-iterations the timed steps decoded: the counters' sum of iterations over valid
    # frames (N per frame when none converges early)
    cw_iters = int(total[2])
    roofline = {"bound": "hbm", "achieved": cn_gbs, "peak": peak, "unit": "GB/s",
                "frac": (cn_gbs / peak) if cn_gbs else None, "traffic": traffic,
                "traffic_production_pass": (dict(traffic_prod, frac=traffic_prod["dram_gbs"] / peak)
                                            if isinstance(traffic_prod, dict) and peak else traffic_prod),
                "kernel": "CN phase: the k_cn_ring launches of one iteration (all degree classes, VN sums fused)",
                "bytes_per_launch": bm["cn"] * min(F, a.lanes),
                "bytes_model": f"2 E_it s_r + 4 (n_1 + n_a) + m/8 per codeword-iteration, s_r = {a.msg_bits // 8} "
                               "(SURVEY 8(d) without the VN write-back, which the fused VN sum keeps in L2), x 64 lanes",
                "peak_source": peak_src,
                "avg_launch_ms": prof_k["cn_ms"] / max(1, prof_k["cn_launches"]), "kernel_timing": kernel_timing,
                "finish_avg_launch_ms": prof_k["vn_ms"] / max(1, prof_k["vn_launches"]),
                # whole timed step: the method's algorithmic floor (SURVEY 8(d) B_alg) x the
                # codeword-iterations decoded, over the device-timed step
                "iteration_alg_frac": (cw_iters * bm["alg"] / (ms_max / 1e3) / 1e9 / peak)}

    # ---- e2e through the host-buffer C-ABI call (pinned host memory, copies inside)
    e2e = None
    if not a.no_e2e:
        v_h = torch.from_numpy(np.tile(v_np, (rep, 1))[:F]).pin_memory()
        xn_h = torch.from_numpy(np.tile(xn_np, (rep, 1))[:F]).pin_memory() if xn_np is not None else None
        sy_h = torch.from_numpy(np.tile(sy_np, (rep, 1))[:F].view(np.int32)).pin_memory()
        out_h = (torch.empty((F, nw), dtype=torch.int32).pin_memory(), torch.empty(F, dtype=torch.int32).pin_memory(),
                 torch.empty(F, dtype=torch.uint8).pin_memory())

        def host_call():
            if a.input == "md":
                dec.decode_md_host(v_h, xn_h, sy_h, a.snr, out=out_h)
            else:
                dec.decode_host(v_h, sy_h, out=out_h)

        host_call()                                                   # warm (allocates staging)
        barrier()
        k_e2e = max(1, min(a.steps, 3))
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            host_call()
        dt = D.max_over_ranks(time.perf_counter() - t0, device=dev)
        W = (st["m"] + 31) // 32
        e2e = {"value": F * world * k_e2e * a.n / dt / 1e6, "unit": "Mb/s",
               "h2d_bytes_per_step": F * world * (a.n * 4 + ((a.n // 8) * 4 if a.input == "md" else 0) + W * 4),
               "d2h_bytes_per_step": F * world * (nw * 4 + 4 + 1),
               "api": ("metldpc_decode_md_host (pinned host buffers; H2D, LLR, decode, D2H inside the call; "
                       if a.input == "md" else
                       "metldpc_decode_host (pinned host LLR / syndrome buffers; H2D, decode, D2H inside the call; ")
                      + ("lane refill: chunked H2D published to the streaming decode's queue"
                         if not (a.no_refill or a.no_et) else "64-lane groups, copies overlapped with decode") + ")",
               "steps": k_e2e, "timing": "host wall clock around the synchronous call, max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = oracle_throughput(a, code, v_np, xn_np, sy_np, a.cpu_budget)

    if rank == 0:
        R = (a.n - st["m"]) / a.n
        conv_frac = counts["converged_timed"] / max(1, counts["frames_timed"])
        out = {
            "metric": METRIC, "value": value, "unit": "Mb/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_max / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": vs_baseline(a, value), "dtype": "f32", "data": "synthetic",
            "value_definition": "n-bit Mb/s: all n decoded bits of every frame per second, converged or not -- "
                                "the paper's Table-1 'Error Correction Speed' n/(N x latency) (P:69-72); "
                                "info_mbps = R x value, goodput_info_mbps = R x n x converged frames / s",
            "config": {"workload": workload_name(a), "code": f"{a.family} stand-in (Table-1 counts), n={a.n}, "
                       f"m={st['m']}, E={st['edges']}, E_it={st['iter_edges']}", "snr": a.snr,
                       "beta": metrics.beta(R, a.snr), "max_iter": a.iters, "early_term": not a.no_et,
                       "rule": a.rule.upper(), "frames_per_gpu": F, "distinct_frames_per_gpu": ND,
                       "lanes_per_group": a.lanes, "groups_in_flight": a.groups, "global_batch": F * world,
                       "msg_bits": a.msg_bits,
                       "lane_refill": not a.no_refill,
                       "l2": f"inputs larger than L2 ({F * a.n * 4 / 1e9:.1f} GB of input per GPU and step, edge "
                             f"messages {st['iter_edges'] * 64 * a.msg_bits / 8 / 1e6:.0f} MB per 64-lane group)",
                       "parallelism": f"dp{world} (frames sharded f mod G; per-step NCCL all-reduce of the FER "
                                      "counters, one all-gather of per-frame results)"},
            "baseline_context": (f"paper Table 1: {paper_mbps(a)} Mb/s (vs_baseline set only for --no-et, the paper's "
                                 f"fixed-N flow; value / paper = {value / paper_mbps(a):.1f}x here): rate "
                                 f"{RATE_COLUMN[a.family][1:]} {'without' if a.no_skip else 'with'} skipping on one TITAN Xp "
                                 "(64 codewords, fixed N iterations) -- context, other hardware")
                                if paper_mbps(a) else None,
            "info_mbps": value * R, "goodput_info_mbps": value * R * conv_frac,
            # the n-bit Mb/s of the same decoding work run as the paper's fixed-N flow (every frame
            # N iterations): value x mean iterations / N
            "fixed_n_equivalent_mbps": value * counts["mean_iters"] / a.iters,
            "input": ("BIAWGN channel LLRs at the SNR (the virtual channel MD reconciliation creates, P:20; "
                      "DESIGN.md R31)" if a.input == "biawgn" else
                      "8-D MD reconciliation output (v, |x|) -> metldpc_llr_from_md (R13) inside the step"),
            **counts,
            "comm": {"backend": "nccl" if world > 1 else None, "world_size": world},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(prof["launches"]), "clocks": clocks,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
