#!/usr/bin/env python
"""Finite-length search over the Table-1-count MET family (DESIGN TOOL for SURVEY 8(f) #4,
not product code): builds candidate codes at n = 10^6 (seeded socket matching, optionally
with 4-cycles among active VNs broken by socket swaps) into the code cache (search_*.npz), and
on a GPU measures their FER / iterations at a few SNRs with the decoder itself (all-GPU frame
generation, MD front end, as tools/fer_sweep.py).

    python tools/met_search.py build            # CPU: write the candidates
    python tools/met_search.py run OUT.jsonl    # GPU: FER of every candidate
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from synth.codes import _CACHE, CODE_SEED, Code, _match, break_4cycles, from_edges  # noqa: E402

OUT = _CACHE


def counts(n, p_inner2):
    """Table-1 counts; p_inner2 n inner checks x2^2 x3 (the rest x2^3 x3)."""
    a, n1, m = n // 8, 7 * n // 8, n - int(round(0.1 * n))
    t2 = int(round(p_inner2 * n))
    e2 = 2 * t2 + 3 * (n1 - t2)
    e1 = int(round(2.8925 * n)) - e2
    a3 = e1 - 2 * a
    assert 0 <= a3 <= a
    core = m - n1
    lo, hi = divmod(e1, core)
    blo, bhi = divmod(e2, a)
    return dict(a=a, n1=n1, m=m, t2=t2, a2=a - a3, a3=a3, core=core, core_deg=(lo, hi), inner_b=(blo, bhi))


def build(n, p_inner2, fix4, seed=CODE_SEED):
    c = counts(n, p_inner2)
    rng = np.random.Generator(np.random.Philox(key=seed))
    a, m, core = c["a"], c["m"], c["core"]
    core_deg_vn = np.concatenate([np.full(c["a2"], 2), np.full(c["a3"], 3)])
    lo, hi = c["core_deg"]
    core_deg_cn = np.concatenate([np.full(core - hi, lo), np.full(hi, lo + 1)])
    inner_deg = np.concatenate([np.full(c["t2"], 2), np.full(c["n1"] - c["t2"], 3)])
    blo, bhi = c["inner_b"]
    inner_per_vn = np.concatenate([np.full(bhi, blo + 1), np.full(a - bhi, blo)])
    v1, c1 = _match(rng, np.repeat(np.arange(a), core_deg_vn), np.repeat(np.arange(core), core_deg_cn), m)
    v2, c2 = _match(rng, np.repeat(np.arange(a), inner_per_vn), np.repeat(np.arange(core, m), inner_deg), m)
    vn = np.concatenate([v1, v2])
    cn = np.concatenate([c1, c2])
    typ = np.concatenate([np.ones(v1.size, np.int8), np.full(v2.size, 2, np.int8)])
    rounds = 0
    if fix4:
        vn, cn, rounds = break_4cycles(vn, cn, typ, rng)
    v3 = np.arange(a, n)
    c3 = rng.permutation(np.arange(core, m))
    vn = np.concatenate([vn, v3])
    cn = np.concatenate([cn, c3])
    pv, pc = rng.permutation(n), rng.permutation(m)
    code = from_edges(n, m, pv[vn], pc[cn], name=f"search_p{p_inner2}_f{int(fix4)}")
    return code, rounds


CANDS = [(p, f) for p in (0.0, 0.025, 0.04375, 0.06) for f in (False, True)]


def cmd_build():
    OUT.mkdir(parents=True, exist_ok=True)
    for p, f in CANDS:
        t = time.time()
        code, rounds = build(10 ** 6, p, f)
        st = code.stats()
        assert (st["m"], st["edges"], st["iter_edges"], st["n_deg1"]) == (900000, 3767500, 2892500, 875000), st
        np.savez(OUT / f"{code.name}.npz", n=code.n, m=code.m, cn_ptr=code.cn_ptr, edge_vn=code.edge_vn,
                 vn_ptr=code.vn_ptr, vn_edge=code.vn_edge)
        print(code.name, "rounds", rounds, f"{time.time() - t:.1f}s", flush=True)


def cmd_run(out_path, snrs=(0.161, 0.165, 0.17, 0.175), frames=512):
    import torch
    from paper_1711_01783_b200 import binding as B
    from paper_1711_01783_b200.build import build as build_lib
    from synth.frames_gpu import gen_batch, pack_bits
    build_lib()
    out = open(out_path, "w")
    for p, f in CANDS:
        name = f"search_p{p}_f{int(f)}"
        z = np.load(OUT / f"{name}.npz")
        code = Code(n=int(z["n"]), m=int(z["m"]), cn_ptr=z["cn_ptr"], edge_vn=z["edge_vn"], vn_ptr=z["vn_ptr"],
                    vn_edge=z["vn_edge"], name=name)
        h = B.Code(code)
        dec = B.Decoder(h, 256, max_iter=100, lane_refill=True)
        for snr in snrs:
            fr = conv = undet = its = 0
            for bi in range(frames // 256):
                x, alpha, u = gen_batch(code.n, 256, snr, 5, bi)
                ub = pack_bits(u)
                sb = dec.syndrome(ub)
                lam = dec.md_alice_llr(x, alpha, snr)
                bits, it, cv = dec.decode(lam, sb)
                err = (bits ^ ub).ne(0).any(-1)
                cvb = cv.bool()
                fr += 256
                conv += int(cvb.sum())
                undet += int((cvb & err).sum())
                its += int(it.sum())
            rec = {"code": name, "p_inner2": p, "fix4": f, "snr": snr, "fer": 1 - conv / fr,
                   "undetected": undet / fr, "mean_iters": its / fr}
            print(json.dumps(rec), flush=True)
            out.write(json.dumps(rec) + "\n")
        dec.close()
        h.close()


if __name__ == "__main__":
    if sys.argv[1] == "build":
        cmd_build()
    else:
        cmd_run(sys.argv[2])
