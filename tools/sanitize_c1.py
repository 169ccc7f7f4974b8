"""C1 decodes for compute-sanitizer (memcheck / racecheck / synccheck): every kernel family of
the path on a tiny code -- LLR init, scatter, the pipelined and tiled CN classes (graph loop
and host-enqueued loop), lane refill waves, the host-buffer streaming path, finalize,
counters, syndrome -- checked against the oracle so a sanitizer run also proves the results.

    compute-sanitizer --tool memcheck python tools/sanitize_c1.py
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import bp  # noqa: E402
from paper_1711_01783_b200 import binding as B  # noqa: E402
from synth.codes import make_met_code  # noqa: E402
from synth.frames import gen_batch, unpack_bits  # noqa: E402


def main():
    code = make_met_code("r0.1", 2048)
    h = B.Code(code)
    fr = gen_batch(code, 0.25, 9, range(70))
    llr = np.stack([bp.llr_from_md_f32(fr["v"][i], fr["xnorm"][i], 0.25) for i in range(70)])
    sy = fr["synd"]
    ref = [bp.decode(code, llr[i], sy[i], 30, prec=32) for i in range(70)]
    L_t, S_t = torch.from_numpy(llr).cuda(), torch.from_numpy(sy.view(np.int32)).cuda()
    modes = [("refill", dict(lane_refill=True)), ("group", dict(lane_refill=False)),
             ("group_k2", dict(lane_refill=False, groups_in_flight=2))]
    if os.environ.get("METLDPC_GRAPH") != "0":
        modes.append(("refill_k2", dict(lane_refill=True, groups_in_flight=2)))
    for name, kw in modes:
        for rule in (B.RULE_EXACT, B.RULE_PHI_LUT):
            dec = B.Decoder(h, 70, rule=rule, max_iter=30, **kw)
            bits, it, cv = dec.decode(L_t, S_t)
            torch.cuda.synchronize()
            bits = bits.cpu().numpy().view(np.uint32)
            for i in range(0, 70, 3):
                o = ref[i] if rule == B.RULE_EXACT else bp.decode(code, llr[i], sy[i], 30, rule=rule, prec=32)
                assert it[i].item() == o["iters"] and np.array_equal(unpack_bits(bits[i], code.n), o["bits"]), (name, i)
            hb, hi, hc = dec.decode_md_host(fr["v"], fr["xnorm"], sy, 0.25)
            assert np.array_equal(hi, it.cpu().numpy()), name
            cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
            dec.counters(it, cv, cnt)
            dec.syndrome(torch.from_numpy(bits.view(np.int32)).cuda())
            torch.cuda.synchronize()
            dec.close()
    print("sanitize_c1: all decodes match the oracle")


if __name__ == "__main__":
    main()
