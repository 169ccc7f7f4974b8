#!/usr/bin/env python
"""Cost of the parts of a refill wave (measurement tool, not product code).

Run once per library variant (METLDPC_LIB=scratch/variants/wrepK/libmetldpc.so, built with
-DMETLDPC_WAVE_REP=K: bit 0 finalize_lanes, 1 scatter, 2 synd launched twice per wave):
    python tools/wave_parts.py NAME EXTRA_LAUNCHES_PER_WAVE OUT.jsonl
Streaming decodes of 1024 r0.1de frames at SNR 0.161 with refill thresholds 1 and 8; the extra
time per wave of a variant over the base is the repeated kernel's cost.
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main(name, extra, out_path):
    import torch
    from paper_1711_01783_b200 import binding as B
    from synth.codes import make_met_code
    from synth.frames_gpu import gen_batch_biawgn, pack_bits
    code = make_met_code("r0.1de", 10 ** 6)
    h = B.Code(code)
    F = 1024
    lam, u = gen_batch_biawgn(code.n, F, 0.161, 9, 0)
    dec0 = B.Decoder(h, 8, max_iter=100)
    sy = dec0.syndrome(pack_bits(u))
    dec0.close()
    out = open(out_path, "a")
    for wmin in (1, 8):
        os.environ["METLDPC_REFILL_MIN"] = str(wmin)
        dec = B.Decoder(h, F, max_iter=100, lane_refill=True)
        dec.decode(lam, sy)
        torch.cuda.synchronize()
        for rep in range(2):
            dec.reset_profile()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            bits, it, cv = dec.decode(lam, sy)
            e1.record()
            torch.cuda.synchronize()
            prof = dec.profile()
            passes = prof["cn_launches"]
            waves = (prof["launches"] - passes * 5) / (5 + extra)
            rec = {"variant": name, "wave_min": wmin, "rep": rep, "ms": e0.elapsed_time(e1), "passes": passes,
                   "waves": waves, "mean_iters": it.float().mean().item()}
            print(json.dumps(rec), flush=True)
            out.write(json.dumps(rec) + "\n")
        dec.close()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3])
