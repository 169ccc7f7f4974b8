#!/usr/bin/env python
"""Device time per pass of the group-mode CUDA-graph loop, fixed N (measurement tool, not product code).

    [METLDPC_LIB=...] python tools/pass_cost.py NAME OUT.jsonl
1024 r0.1de frames (16 groups of 64, one in flight), N = 100, ET off: time / 1600 passes.
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main(name, out_path):
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
    dec = B.Decoder(h, F, max_iter=100, early_term=False, lane_refill=False)
    dec.decode(lam, sy)
    torch.cuda.synchronize()
    out = open(out_path, "a")
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dec.decode(lam, sy)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        rec = {"variant": name, "rep": rep, "ms": ms, "passes": F // 64 * 100, "t_pass_ms": ms / (F // 64 * 100)}
        print(json.dumps(rec), flush=True)
        out.write(json.dumps(rec) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
