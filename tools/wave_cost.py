#!/usr/bin/env python
"""Cost of one lane-refill wave and of one streaming pass (measurement tool, not product code).

Runs on the headline code (r0.1de, n = 10^6, BIAWGN frames):
  1. group mode, fixed N: device time per pass (t_group);
  2. streaming decodes at several SNRs / refill thresholds: passes and waves from the device
     counters (metldpc_get_profile), device time; least squares time = passes t_pass + waves W.
    python tools/wave_cost.py OUT.jsonl
"""
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main(out_path):
    import torch
    from paper_1711_01783_b200 import binding as B
    from paper_1711_01783_b200.build import build
    from synth.codes import make_met_code
    from synth.frames_gpu import gen_batch_biawgn, pack_bits
    build()
    code = make_met_code("r0.1de", 10 ** 6)
    h = B.Code(code)
    out = open(out_path, "w")
    F = 1024

    def frames(snr):
        lam, u = gen_batch_biawgn(code.n, F, snr, 9, 0)
        dec0 = B.Decoder(h, 8, max_iter=100)
        sy = dec0.syndrome(pack_bits(u))
        dec0.close()
        return lam, sy

    def timed(dec, lam, sy):
        dec.decode(lam, sy)
        torch.cuda.synchronize()
        dec.reset_profile()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        bits, it, cv = dec.decode(lam, sy)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), dec.profile(), it.float().mean().item(), cv.float().mean().item()

    lam, sy = frames(0.161)
    dec = B.Decoder(h, F, max_iter=100, early_term=False)
    ms, prof, mi, cv = timed(dec, lam, sy)
    t_group = ms / (F // 64 * 100)
    dec.close()
    rec = {"mode": "group fixed N", "ms": ms, "passes": F // 64 * 100, "t_pass_ms": t_group}
    print(json.dumps(rec), flush=True)
    out.write(json.dumps(rec) + "\n")
    rows = []
    for snr in (0.161, 0.2, 0.3):
        lam, sy = frames(snr)
        for wmin in (1, 4, 8, 16, 64):
            os.environ["METLDPC_REFILL_MIN"] = str(wmin)
            dec = B.Decoder(h, F, max_iter=100, lane_refill=True)
            ms, prof, mi, cv = timed(dec, lam, sy)
            passes = prof["cn_launches"]
            # launches = passes * (classes + 2) + waves * 5 (since the loop control rides on the latch)
            ncls = 3
            waves = (prof["launches"] - passes * (ncls + 2)) / 5
            rec = {"mode": "stream", "snr": snr, "wave_min": wmin, "ms": ms, "passes": passes, "waves": waves,
                   "mean_iters": mi, "converged": cv}
            rows.append((passes, waves, ms))
            print(json.dumps(rec), flush=True)
            out.write(json.dumps(rec) + "\n")
            dec.close()
    A = np.array([[p, w] for p, w, _ in rows], float)
    y = np.array([m for _, _, m in rows])
    (t_pass, W), *_ = np.linalg.lstsq(A, y, rcond=None)
    rec = {"fit": "ms = passes t_pass + waves W", "t_pass_ms": t_pass, "wave_ms": W, "t_group_ms": t_group}
    print(json.dumps(rec), flush=True)
    out.write(json.dumps(rec) + "\n")


if __name__ == "__main__":
    main(sys.argv[1])
