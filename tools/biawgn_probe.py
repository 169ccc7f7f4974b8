"""Probe: FER of a search candidate on the plain BIAWGN channel (all-zero word) vs the MD front end (design tool)."""
import sys, json, numpy as np, torch
sys.path.insert(0, '.')
from tools.met_search import build, OUT
from synth.codes import Code
from paper_1711_01783_b200 import binding as B
from paper_1711_01783_b200.build import build as build_lib
build_lib()
import os
name = "search_p0.06_f1"
p = OUT / f"{name}.npz"
if not p.exists():
    code, _ = build(10**6, 0.06, True)
    np.savez(p, n=code.n, m=code.m, cn_ptr=code.cn_ptr, edge_vn=code.edge_vn, vn_ptr=code.vn_ptr, vn_edge=code.vn_edge)
z = np.load(p)
code = Code(n=int(z["n"]), m=int(z["m"]), cn_ptr=z["cn_ptr"], edge_vn=z["edge_vn"], vn_ptr=z["vn_ptr"], vn_edge=z["vn_edge"])
h = B.Code(code)
dec = B.Decoder(h, 256, max_iter=int(sys.argv[2]) if len(sys.argv) > 2 else 100, lane_refill=True)
g = torch.Generator(device="cuda"); g.manual_seed(1)
W = (code.m + 31) // 32
out = open(sys.argv[1], "w")
for snr in [0.155, 0.16, 0.165, 0.17]:
    conv = its = 0
    for b in range(2):
        lam = (2 * snr + 2 * np.sqrt(snr) * torch.randn(256, code.n, device="cuda", generator=g)).float()
        sy = torch.zeros(256, W, dtype=torch.int32, device="cuda")
        bits, it, cv = dec.decode(lam, sy)
        conv += int(cv.sum()); its += int(it.sum())
    rec = {"code": name, "channel": "BIAWGN N(2s,4s), all-zero word", "snr": snr, "fer": 1 - conv / 512, "mean_iters": its / 512, "max_iter": dec.cfg.max_iter}
    print(json.dumps(rec), flush=True); out.write(json.dumps(rec) + "\n")
