#!/usr/bin/env python
"""Figure-2 analogue: decoding speed and latency vs the number of
codewords decoded in parallel, fixed N iterations (the paper's flow, early_term = 0).

    python tools/batch_sweep.py [--family r0.1 --n 1000000 --iters 100 --snr 0.161]
                                [--batches 1,2,4,...,512] [--out profiles/r1_fig2_sweep.jsonl]

Speed = frames * n / device time (Table-1 convention); latency per iteration per codeword
= time / (N * frames) (Table 1 note 3).
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--family", default="r0.1")
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--snr", type=float, default=0.161)
    ap.add_argument("--batches", default="1,2,4,8,16,32,64,128,256,512")
    ap.add_argument("--groups", type=int, default=4)
    ap.add_argument("--rule", choices=["exact", "lut"], default="exact")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()

    import torch
    from paper_1711_01783_b200 import binding as B
    from paper_1711_01783_b200.build import build
    from synth.codes import make_met_code
    from synth.frames_gpu import gen_batch, pack_bits

    build()
    code = make_met_code(a.family, a.n)
    h = B.Code(code)
    bmax = max(int(b) for b in a.batches.split(","))
    x, alpha, u = gen_batch(a.n, bmax, a.snr, 3, 0)
    dec0 = B.Decoder(h, bmax, groups_in_flight=1)
    sb = dec0.syndrome(pack_bits(u))
    lam = dec0.md_alice_llr(x, alpha, a.snr)
    del x, alpha, u
    out = open(a.out, "w") if a.out else None
    for b in [int(v) for v in a.batches.split(",")]:
        dec = B.Decoder(h, b, rule=0 if a.rule == "exact" else 1, max_iter=a.iters, early_term=False,
                        groups_in_flight=a.groups)
        res = dec.decode(lam[:b], sb[:b])
        torch.cuda.synchronize()
        ms = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dec.decode(lam[:b], sb[:b], out=res)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        t = min(ms) / 1e3
        rec = {"experiment": "fig2_batch_sweep", "family": a.family, "n": a.n, "iters": a.iters, "codewords": b,
               "groups_in_flight": min(a.groups, (b + 63) // 64), "rule": a.rule.upper(),
               "speed_mbps": b * a.n / t / 1e6, "latency_ms": t * 1e3,
               "latency_per_iter_per_codeword_ms": t * 1e3 / (a.iters * b)}
        print(json.dumps(rec), flush=True)
        if out:
            out.write(json.dumps(rec) + "\n")
        dec.close()


if __name__ == "__main__":
    main()
