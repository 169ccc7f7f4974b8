"""CPU test of bench.py's output contract through its reference arm (the oracle on host
cores, no GPU): one JSON line with the keys the driver reads."""
import json
import subprocess
import sys


def test_reference_arm_json_line(root):
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--n", "2048", "--steps", "1",
                          "--warmup", "0", "--frames", "8", "--distinct", "8", "--cpu-budget", "1"],
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "Mb/s" and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("custom")          # n != 10^6 is not a named workload
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
