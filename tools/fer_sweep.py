#!/usr/bin/env python
"""C5 (BASELINE configs[4]): FER / iteration sweep over SNR with MD-reconciliation input.

For each SNR the whole reverse-reconciliation chain runs on the GPU: seeded frames
(synth/frames_gpu.py) -> Bob's syndrome S_B = H u (metldpc_syndrome, Step 1) -> Alice's
LLRs from (x, alpha) (metldpc_md_alice_llr, R13/N6) -> syndrome BP with per-frame early
termination (metldpc_decode) -> FER (non-converged frames), undetected errors (converged,
c != u), mean iterations, iteration histogram, device-timed decode throughput.

    python tools/fer_sweep.py [--family r0.1] [--n 1000000] [--frames 512] [--iters 100]
                              [--snrs 0.14,0.15,...] [--out profiles/r1_fer_sweep.jsonl]
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--family", default="r0.1de")
    ap.add_argument("--channel", choices=["md", "biawgn"], default="md",
                    help="md: the MD reconciliation chain on the GPU; biawgn: channel LLRs N(+-2s, 4s) (R31)")
    ap.add_argument("--msg-bits", type=int, choices=[32, 16], default=32)
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--frames", type=int, default=512)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--snrs", default="0.14,0.15,0.16,0.161,0.17,0.175,0.18,0.19,0.20")
    ap.add_argument("--rule", choices=["exact", "lut"], default="exact")
    ap.add_argument("--key", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--groups", type=int, default=1, help="lane groups in flight")
    ap.add_argument("--no-refill", action="store_true", help="group mode instead of lane refill")
    a = ap.parse_args()

    import torch
    from paper_1711_01783_b200 import binding as B
    from paper_1711_01783_b200 import metrics
    from paper_1711_01783_b200.build import build
    from synth.codes import make_met_code
    from synth.frames_gpu import gen_batch, gen_batch_biawgn, pack_bits

    build()
    code = make_met_code(a.family, a.n)
    st = code.stats()
    R = (st["n"] - st["m"]) / st["n"]
    h = B.Code(code)
    dec = B.Decoder(h, a.batch, rule=0 if a.rule == "exact" else 1, max_iter=a.iters, groups_in_flight=a.groups,
                    lane_refill=not a.no_refill, msg_bits=a.msg_bits)
    out = open(a.out, "w") if a.out else None
    for snr in [float(s) for s in a.snrs.split(",")]:
        frames = conv = undet = iters_sum = 0
        hist = [0] * (a.iters + 1)
        dev_ms = 0.0
        for bi in range((a.frames + a.batch - 1) // a.batch):
            nb = min(a.batch, a.frames - bi * a.batch)
            if a.channel == "md":
                x, alpha, u = gen_batch(a.n, nb, snr, a.key, bi)
            else:
                lam, u = gen_batch_biawgn(a.n, nb, snr, a.key, bi)
            ub = pack_bits(u)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sb = dec.syndrome(ub)                      # Bob, Step 1
            if a.channel == "md":
                lam = dec.md_alice_llr(x, alpha, snr)  # Alice, MD front end
            bits, it, cv = dec.decode(lam, sb)
            e1.record()
            torch.cuda.synchronize()
            dev_ms += e0.elapsed_time(e1)
            err = (bits ^ ub)
            nerr = torch.zeros(nb, dtype=torch.int64, device=bits.device)
            for sh in range(32):
                nerr += ((err >> sh) & 1).sum(-1)
            cvb = cv.bool()
            frames += nb
            conv += int(cvb.sum())
            undet += int((cvb & (nerr > 0)).sum())
            itc = it.cpu().tolist()
            iters_sum += sum(itc)
            for v in itc:
                hist[min(max(v, 0), a.iters)] += 1
        rec = {"config": "C5", "family": a.family, "channel": a.channel, "msg_bits": a.msg_bits, "n": a.n,
               "snr": snr, "beta": metrics.beta(R, snr),
               "max_iter": a.iters, "rule": a.rule.upper(), "batch": a.batch, "groups": a.groups,
               "lane_refill": not a.no_refill, "frames": frames, "fer": 1.0 - conv / frames,
               "undetected_rate": undet / frames, "mean_iters": iters_sum / frames,
               "decode_mbps": frames * a.n / (dev_ms / 1e3) / 1e6,
               "iter_hist": {str(k): v for k, v in enumerate(hist) if v}}
        print(json.dumps(rec), flush=True)
        if out:
            out.write(json.dumps(rec) + "\n")
            out.flush()


if __name__ == "__main__":
    main()
