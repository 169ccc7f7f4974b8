"""Debug helper (not product code): decode C1 / a random code under the current env switches."""
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
from oracle import bp
from paper_1711_01783_b200 import binding as B
from synth.codes import make_met_code, random_code
from synth.frames import gen_batch, unpack_bits
codes = {"c1": lambda: make_met_code("r0.1", 2048),
         "rand": lambda: random_code(600, 240, np.random.default_rng(11), frac_deg1=0.3, act_deg=(2, 5))}
import os
keep = []
for which in sys.argv[2].split(","):
    code = codes[which]()
    h = B.Code(code)
    fr = gen_batch(code, 0.3, 5, range(40))
    llr = np.stack([bp.llr_from_md_f32(fr["v"][i], fr["xnorm"][i], 0.3) for i in range(40)])
    rules = [int(x) for x in os.environ.get("RULES", "0,1").split(",")]
    msgs = [int(x) for x in os.environ.get("MSGS", "32,16").split(",")]
    refill = os.environ.get("REFILL", "1") == "1"
    for rule in rules:
        for msg in msgs:
            print("start", which, rule, msg, flush=True)
            dec = B.Decoder(h, 40, rule=rule, max_iter=30, msg_bits=msg, lane_refill=refill)
            bits, it, cv = dec.decode(torch.from_numpy(llr).cuda(), torch.from_numpy(fr["synd"].view(np.int32)).cuda())
            torch.cuda.synchronize()
            print("decoded", which, rule, msg, it[:8].tolist(), flush=True)
            if os.environ.get("KEEP"):
                keep.append((h, dec))
