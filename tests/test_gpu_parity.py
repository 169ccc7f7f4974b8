"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE north_star): hard decisions, iteration counts
and converged flags bit-exact against the fp32 replay M3; messages bit-exact
against M3 every iteration, and M3 is within 1e-3 max(1,|LLR|) of a
teacher-forced fp64 step (tests/test_oracle.py), so the GPU is too.
Inputs are seeded synthetic frames from synth/ (never from the CUDA path).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import bp  # noqa: E402
from paper_1711_01783_b200 import binding as B  # noqa: E402
from synth.codes import from_dense, make_met_code, random_code, write_alist  # noqa: E402
from synth.frames import gen_batch, pack_bits, unpack_bits  # noqa: E402

RULES = [B.RULE_EXACT, B.RULE_PHI_LUT]


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1711_01783_b200.build import build
    build()


def _frames(code, snrs, key=0):
    """Batch with frames at several SNRs (mix of converging and failing frames)."""
    parts = [gen_batch(code, s, key, range(i * 1000, i * 1000 + k)) | {"snr": np.full(k, s)}
             for i, (s, k) in enumerate(snrs)]
    out = {k: np.concatenate([p[k] for p in parts]) for k in ("u", "v", "xnorm", "synd", "snr")}
    return out


def _llr_oracle(fr):
    return np.stack([bp.llr_from_md_f32(fr["v"][i], fr["xnorm"][i], fr["snr"][i]) for i in range(len(fr["v"]))])


def _gpu_decode(code_h, llr, synd, rule, max_iter, et=True, lanes=64, max_batch=None, groups=None, refill=None):
    dec = B.Decoder(code_h, max_batch or llr.shape[0], rule=rule, max_iter=max_iter, early_term=et,
                    lanes_per_group=lanes, groups_in_flight=groups, lane_refill=refill)
    bits, iters, conv = dec.decode(torch.from_numpy(llr).cuda(), torch.from_numpy(synd.view(np.int32)).cuda())
    torch.cuda.synchronize()
    return dec, bits.cpu().numpy().view(np.uint32), iters.cpu().numpy(), conv.cpu().numpy()


def _assert_frame_equal(code, o, bits_row, it, cv, tag=""):
    ob = bp.decode  # noqa
    assert it == o["iters"], (tag, it, o["iters"])
    assert bool(cv) == o["converged"], tag
    assert np.array_equal(unpack_bits(bits_row, code.n), o["bits"]), tag


@pytest.fixture(scope="module")
def c1():
    code = make_met_code("r0.1", 2048)
    return code, B.Code(code)


# ----------------------------------------------------------------------------- LLR init (a1)

@pytest.mark.parametrize("with_norm", [True, False])
def test_llr_from_md_bit_exact(c1, with_norm):
    code, h = c1
    fr = _frames(code, [(0.161, 3), (0.3, 2)])
    dec = B.Decoder(h, 8)
    v = torch.from_numpy(fr["v"]).cuda()
    out = torch.empty_like(v)
    xn = torch.from_numpy(fr["xnorm"]).cuda() if with_norm else None
    for i in range(len(fr["v"])):
        B.metldpc_llr_from_md(dec.h, 1, 8, float(fr["snr"][i]), v[i:i + 1], None if xn is None else xn[i:i + 1],
                              out[i:i + 1])
    got = out.cpu().numpy()
    for i in range(len(fr["v"])):
        ref = bp.llr_from_md_f32(fr["v"][i], fr["xnorm"][i] if with_norm else None, fr["snr"][i])
        assert np.array_equal(got[i].view(np.uint32), ref.view(np.uint32))


# ----------------------------------------------------------------------------- full decode vs M3

@pytest.mark.parametrize("rule", RULES)
def test_c1_bits_iters_flags_bit_exact(c1, rule):
    """C1 (BASELINE configs[0]): n=2048 rate 0.1, SNR 0.161 (4 frames) plus frames at
    0.2/0.3/0.5 so early termination fires at many different iterations."""
    code, h = c1
    fr = _frames(code, [(0.161, 4), (0.2, 4), (0.3, 4), (0.5, 4)])
    llr = _llr_oracle(fr)
    _, bits, iters, conv = _gpu_decode(h, llr, fr["synd"], rule, 100)
    nconv = 0
    for i in range(len(llr)):
        o = bp.decode(code, llr[i], fr["synd"][i], 100, early_term=True, rule=rule, prec=32)
        _assert_frame_equal(code, o, bits[i], iters[i], conv[i], f"frame {i}")
        nconv += o["converged"]
    assert 4 <= nconv < len(llr)      # both regimes exercised


@pytest.mark.parametrize("rule", RULES)
def test_c1_messages_every_iteration(c1, rule):
    """r^l and L^l bit-identical to the oracle's trace for l = 1..N (ET off), for lanes in both
    halves of the pair rows (lanes t and t + 32 share a 64-bit accumulator word, N3)."""
    code, h = c1
    fr = _frames(code, [(0.161, 18), (0.3, 18)])
    llr = _llr_oracle(fr)
    lanes = (0, 1, 17, 18, 32, 33, 34, 35)   # frame i decodes in lane i
    N = 40
    traces = {i: bp.decode(code, llr[i], fr["synd"][i], N, early_term=False, rule=rule, prec=32, trace=True)
              for i in lanes}
    dec = B.Decoder(h, len(llr), rule=rule, max_iter=N, early_term=False)
    L_t = torch.from_numpy(llr).cuda()
    S_t = torch.from_numpy(fr["synd"].view(np.int32)).cuda()
    for l in range(1, N + 1):
        dec.decode(L_t, S_t, max_iter=l)
        for i in lanes:
            r, L = dec.dump(i)
            assert np.array_equal(r.view(np.uint32), traces[i]["r_trace"][l - 1].view(np.uint32)), (l, i)
            assert np.array_equal(L.view(np.uint32), traces[i]["L_trace"][l - 1].view(np.uint32)), (l, i)


@pytest.mark.parametrize("rule", RULES)
def test_no_skip_variant_bit_exact(c1, rule):
    """Table 1 "without skipping" (METLDPC_CODE_NO_SKIP, R26): degree-1 VNs are
    iterated, every inner CN becomes a (4,0) class; bits/iterations/flags bit-exact against
    the oracle's no-skip replay, and messages of every edge bit-exact after 7 iterations."""
    code, _ = c1
    h = B.Code(code, no_skip=True)
    assert (h.info.n_active, h.info.n_deg1, h.info.iter_edges) == (code.n, 0, code.num_edges)
    fr = _frames(code, [(0.161, 4), (0.2, 4), (0.3, 4), (0.5, 4)])
    llr = _llr_oracle(fr)
    dec, bits, iters, conv = _gpu_decode(h, llr, fr["synd"], rule, 100)
    nconv = 0
    for i in range(len(llr)):
        o = bp.decode(code, llr[i], fr["synd"][i], 100, early_term=True, rule=rule, prec=32, no_skip=True)
        _assert_frame_equal(code, o, bits[i], iters[i], conv[i], f"frame {i}")
        nconv += o["converged"]
    assert 4 <= nconv < len(llr)
    dec = B.Decoder(h, len(llr), rule=rule, max_iter=7, early_term=False)
    dec.decode(torch.from_numpy(llr).cuda(), torch.from_numpy(fr["synd"].view(np.int32)).cuda())
    for i in (0, 9):
        o = bp.decode(code, llr[i], fr["synd"][i], 7, early_term=False, rule=rule, prec=32, trace=True, no_skip=True)
        r, L = dec.dump(i)
        assert np.array_equal(r.view(np.uint32), o["r_trace"][-1].view(np.uint32)), i
        assert np.array_equal(L.view(np.uint32), o["L_trace"][-1].view(np.uint32)), i


@pytest.mark.parametrize("et", [True, False])
def test_batch_lane_and_group_invariance(c1, et):
    """S:220 / R12: a frame's result does not depend on batch size, lane, group size or
    lane refill (streaming decode vs group mode)."""
    code, h = c1
    fr = _frames(code, [(0.161, 30), (0.3, 40), (0.6, 30)])
    llr = _llr_oracle(fr)
    ref = None
    for lanes, groups, refill in ((32, 1, None), (64, 1, False), (64, 1, True), (64, 2, True), (64, 3, False),
                                  (128, 2, None)):
        for order in ("fwd", "rev"):
            idx = np.arange(len(llr)) if order == "fwd" else np.arange(len(llr))[::-1].copy()
            _, bits, iters, conv = _gpu_decode(h, llr[idx], fr["synd"][idx], B.RULE_EXACT, 60, et=et, lanes=lanes,
                                               groups=groups, refill=refill)
            inv = np.argsort(idx)
            res = (bits[inv], iters[inv], conv[inv])
            if ref is None:
                ref = res
            else:
                for a, b in zip(ref, res):
                    assert np.array_equal(a, b), (lanes, groups, refill, order)
    # single-frame batches agree too
    for i in (0, 45, 99):
        _, bits, iters, conv = _gpu_decode(h, llr[i:i + 1], fr["synd"][i:i + 1], B.RULE_EXACT, 60, et=et)
        assert np.array_equal(bits[0], ref[0][i]) and iters[0] == ref[1][i] and conv[0] == ref[2][i]


def test_ragged_batch_max_batch_and_host_path(c1):
    """Ragged lane counts (batch % 32 != 0), batch < max_batch, and decode_host (host
    buffers, pipelined copies) give the device-path results."""
    code, h = c1
    fr = _frames(code, [(0.2, 37), (0.4, 40)])
    llr = _llr_oracle(fr)
    _, bits, iters, conv = _gpu_decode(h, llr, fr["synd"], B.RULE_PHI_LUT, 50, max_batch=200, groups=1)
    dec = B.Decoder(h, 200, rule=B.RULE_PHI_LUT, max_iter=50, groups_in_flight=2)
    hb, hi, hc = dec.decode_host(np.ascontiguousarray(llr), np.ascontiguousarray(fr["synd"]))
    assert np.array_equal(hb, bits) and np.array_equal(hi, iters) and np.array_equal(hc, conv)
    for i in (0, 36, 76):
        o = bp.decode(code, llr[i], fr["synd"][i], 50, rule=B.RULE_PHI_LUT, prec=32)
        _assert_frame_equal(code, o, bits[i], iters[i], conv[i])


@pytest.mark.parametrize("rule,groups,wave", [(B.RULE_EXACT, 2, "16"), (B.RULE_PHI_LUT, 1, "1"), (B.RULE_EXACT, 3, "40")])
def test_lane_refill_streaming_bit_exact(c1, rule, groups, wave, monkeypatch):
    """Lane refill (metldpc_config_t.lane_refill, streaming decode): 301 frames (a ragged
    batch: 4 x 64 + 45) at SNRs from 0.16 to 0.6, so lanes latch at very different
    iterations and are refilled from the queue while others iterate; one frame has a
    non-finite LLR and one is noiseless.  Every frame's bits, iteration count and flag equal
    the oracle's and the group-mode decode's, for several refill thresholds."""
    monkeypatch.setenv("METLDPC_REFILL_MIN", wave)
    code, h = c1
    fr = _frames(code, [(0.16, 60), (0.2, 80), (0.3, 80), (0.6, 81)], key=11)
    llr = _llr_oracle(fr)
    llr[5, 100] = np.nan
    llr[7] = ((1.0 - 2.0 * fr["u"][7]) * 8.0).astype(np.float32)
    nb = llr.shape[0]
    dec = B.Decoder(h, nb, rule=rule, max_iter=60, groups_in_flight=groups, lane_refill=True)
    bits, iters, conv = dec.decode(torch.from_numpy(llr).cuda(), torch.from_numpy(fr["synd"].view(np.int32)).cuda())
    torch.cuda.synchronize()
    bits, iters, conv = bits.cpu().numpy().view(np.uint32), iters.cpu().numpy(), conv.cpu().numpy()
    _, gb, gi, gc = _gpu_decode(h, llr, fr["synd"], rule, 60, groups=groups, refill=False)
    assert np.array_equal(bits, gb) and np.array_equal(iters, gi) and np.array_equal(conv, gc)
    assert iters[5] == -1 and conv[5] == 0 and not bits[5].any()
    assert iters[7] == 1 and conv[7] == 1
    assert len(set(iters.tolist())) > 10          # lanes really latch at many different iterations
    for i in list(range(0, nb, 7)) + [nb - 1]:
        if i == 5:
            continue
        o = bp.decode(code, llr[i], fr["synd"][i], 60, early_term=True, rule=rule, prec=32)
        _assert_frame_equal(code, o, bits[i], iters[i], conv[i], f"frame {i}")


def test_lane_refill_edge_cases(c1):
    """Streaming decode corner cases: fewer frames than lanes, max_iter = 1 (every frame's
    final test is its second pass), and a queue of noiseless frames that all latch at l = 1
    so every lane is refilled every other pass; each against group mode."""
    code, h = c1
    fr = _frames(code, [(0.25, 140)], key=23)
    llr = _llr_oracle(fr)
    clean = ((1.0 - 2.0 * fr["u"]) * 8.0).astype(np.float32)
    for x, nf, N in ((llr, 5, 40), (llr, 140, 1), (clean, 140, 30)):
        a = _gpu_decode(h, x[:nf], fr["synd"][:nf], B.RULE_EXACT, N, refill=True, groups=2)[1:]
        b = _gpu_decode(h, x[:nf], fr["synd"][:nf], B.RULE_EXACT, N, refill=False, groups=2)[1:]
        for u, v in zip(a, b):
            assert np.array_equal(u, v), (nf, N)
    _, bits, iters, conv = _gpu_decode(h, clean, fr["synd"], B.RULE_EXACT, 30, refill=True)
    assert (iters == 1).all() and conv.all()
    for i in range(0, 140, 13):
        assert np.array_equal(unpack_bits(bits[i], code.n), fr["u"][i])


def test_edge_cases(c1):
    """Zero noise -> l = 1, c = u; non-finite LLR -> iterations -1 (R24) without
    disturbing neighbours; max_iter = 1; empty batch."""
    code, h = c1
    fr = _frames(code, [(0.3, 4)])
    llr = _llr_oracle(fr)
    clean = ((1.0 - 2.0 * fr["u"][0]) * 8.0).astype(np.float32)
    llr2 = np.stack([clean, llr[1], llr[2], llr[3]])
    llr2[2, 77] = np.inf
    _, bits, iters, conv = _gpu_decode(h, llr2, fr["synd"], B.RULE_EXACT, 100)
    assert iters[0] == 1 and conv[0] == 1 and np.array_equal(unpack_bits(bits[0], code.n), fr["u"][0])
    assert iters[2] == -1 and conv[2] == 0 and not bits[2].any()
    for i in (1, 3):
        o = bp.decode(code, llr2[i], fr["synd"][i], 100, prec=32)
        _assert_frame_equal(code, o, bits[i], iters[i], conv[i])
    _, bits, iters, conv = _gpu_decode(h, llr, fr["synd"], B.RULE_EXACT, 1)
    for i in range(4):
        o = bp.decode(code, llr[i], fr["synd"][i], 1, prec=32)
        _assert_frame_equal(code, o, bits[i], iters[i], conv[i])
    dec = B.Decoder(h, 4)
    B.metldpc_decode(dec.h, 0, None, None, 0, None, None, None)   # empty batch is a no-op


def test_generic_degree_paths_and_alist(tmp_path):
    """Random codes exercising every CN-degree window (0-4, 5-8, 9-12, 13-16, 17-32),
    loaded through alist, against the oracle."""
    rng = np.random.default_rng(21)
    windows = set()
    for t, (n, m, deg) in enumerate([(60, 20, (2, 3)), (80, 12, (2, 4)), (120, 12, (2, 3)), (90, 16, (2, 3))]):
        for _ in range(100):
            code = random_code(n, m, rng, frac_deg1=0.3, act_deg=deg)
            if code.cn_degree.max() <= 32:
                break
        p = tmp_path / f"c{t}.alist"
        write_alist(code, p)
        h = B.Code(alist=str(p))
        windows.update(int(np.searchsorted([4, 8, 12, 16, 32], d)) for d in code.cn_degree)
        assert h.info.edges == code.num_edges and h.info.max_cn_deg == code.cn_degree.max()
        u = rng.integers(0, 2, n).astype(np.uint8)
        s = (code.dense().astype(int) @ u) % 2
        llr = ((1 - 2.0 * u) * rng.uniform(0.2, 2.5, (8, n))).astype(np.float32)
        llr[:, :5] *= -1
        synd = np.stack([pack_bits(s)] * 8)
        for rule in RULES:
            _, bits, iters, conv = _gpu_decode(h, llr, synd, rule, 30)
            for i in range(8):
                o = bp.decode(code, llr[i], synd[i], 30, rule=rule, prec=32)
                _assert_frame_equal(code, o, bits[i], iters[i], conv[i], f"code {t} frame {i}")
    assert windows == {0, 1, 2, 3, 4}, windows


def _degree1_edge_code():
    """CN 0, 1: VNs 0-2 (active) + one degree-1 VN each -> the (3,1) pipelined class;
    CN 2: VN 0 + two degree-1 VNs -> the generic class; CN 3: VNs 1, 2 + VN 0."""
    h = np.zeros((4, 8), np.uint8)
    h[0, [0, 1, 2, 3]] = 1
    h[1, [0, 1, 2, 4]] = 1
    h[2, [0, 5, 6]] = 1
    h[3, [0, 1, 2, 7]] = 1
    return from_dense(h)


@pytest.mark.parametrize("rule", RULES)
def test_degree1_decision_edge_cases(rule):
    """Degree-1 decisions (N1, R27) through the pipelined and the generic CN kernels, bit-exact
    against M3 on crafted priors: signed zeros, exact ties, |lambda| around the 30 clamp and far
    beyond the phi table, tiny values; 1-4 iterations, ET on and off."""
    code = _degree1_edge_code()
    hd = B.Code(code)
    rng = np.random.default_rng(27)
    special = np.array([0.0, -0.0, 30.5, -30.5, 31.0, -29.9, 32.0, 64.0, -70.0, 1e6, -1e6, 1e-30, -1e-30,
                        0.5, -0.5, 3.0], np.float32)
    n = code.n
    llr = rng.choice(special, size=(64, n)).astype(np.float32)
    llr[32:] = rng.normal(0.0, 4.0, (32, n)).astype(np.float32)
    llr[40:44, :3] = 32.0                     # inputs whose CN output exceeds the clamp
    llr[40:44, 3] = np.float32(-30.5)
    llr[44:48, 3] = -llr[44:48, 0]            # ties between a prior and a message
    synd = np.stack([pack_bits(rng.integers(0, 2, code.m)) for _ in range(64)])
    for et in (True, False):
        for it in (1, 2, 4):
            _, bits, iters, conv = _gpu_decode(hd, llr, synd, rule, it, et=et)
            for i in range(64):
                o = bp.decode(code, llr[i], synd[i], it, early_term=et, rule=rule, prec=32)
                _assert_frame_equal(code, o, bits[i], iters[i], conv[i], f"frame {i} N {it} et {et}")


def test_empty_check_row():
    """A degree-0 CN with S_B bit 1 can never be satisfied (R23)."""
    h = np.array([[1, 1, 0, 0], [0, 1, 1, 1], [0, 0, 0, 0]], np.uint8)
    code = from_dense(h)
    hd = B.Code(code)
    llr = np.array([[2.0, 1.0, -1.5, 0.7]] * 2, np.float32)
    synd = np.stack([pack_bits([0, 0, 0]), pack_bits([0, 0, 1])])
    _, bits, iters, conv = _gpu_decode(hd, llr, synd, B.RULE_EXACT, 10)
    for i in range(2):
        o = bp.decode(code, llr[i], synd[i], 10, prec=32)
        _assert_frame_equal(code, o, bits[i], iters[i], conv[i])
    assert conv[1] == 0


# ----------------------------------------------------------------------------- larger configs

def test_c2_sampled_lanes():
    """C2 (configs[1]): n=65,536, 64-codeword batch at SNR 0.161 + 0.2; lanes
    0, 17, 38, 63 replayed by the oracle bit-exactly; every converged lane
    satisfies H c = S_B."""
    code = make_met_code("r0.1", 65536)
    h = B.Code(code)
    fr = _frames(code, [(0.161, 40), (0.2, 24)])
    llr = _llr_oracle(fr)
    _, bits, iters, conv = _gpu_decode(h, llr, fr["synd"], B.RULE_EXACT, 100)
    for i in (0, 17, 38, 63):
        o = bp.decode(code, llr[i], fr["synd"][i], 100, prec=32)
        _assert_frame_equal(code, o, bits[i], iters[i], conv[i], f"lane {i}")
    for i in np.flatnonzero(conv):
        s = unpack_bits(fr["synd"][i], code.m)
        assert np.array_equal(bp.syndrome(code, unpack_bits(bits[i], code.n)), s)


@pytest.mark.parametrize("rule", RULES)
def test_c3_full_size_sampled_lane(rule):
    """C3 at BASELINE's full size (n = 10^6, rate 0.1, SNR 0.161, N = 100) in the bench's
    launch configuration (64-lane groups, two groups): two sampled lanes (one per group)
    replayed by the oracle bit-exactly."""
    code = make_met_code("r0.1", 10 ** 6)
    h = B.Code(code)
    nf = 72
    fr = gen_batch(code, 0.161, 0, range(nf))
    dec = B.Decoder(h, nf, rule=rule, max_iter=100)
    v = torch.from_numpy(fr["v"]).cuda()
    xn = torch.from_numpy(fr["xnorm"]).cuda()
    llr_d = dec.llr_from_md(v, xn, 0.161)
    bits, iters, conv = dec.decode(llr_d, torch.from_numpy(fr["synd"].view(np.int32)).cuda())
    bits = bits.cpu().numpy().view(np.uint32)
    iters = iters.cpu().numpy()
    conv = conv.cpu().numpy()
    for i in (5, 70):
        lam = bp.llr_from_md_f32(fr["v"][i], fr["xnorm"][i], 0.161)
        o = bp.decode(code, lam, fr["synd"][i], 100, rule=rule, prec=32)
        _assert_frame_equal(code, o, bits[i], iters[i], conv[i], f"lane {i}")
    assert (iters > 0).all()


def test_c4_rate005_full_size_sampled_lane():
    """C4 (configs[3]): rate-0.05 stand-in (Table-1 counts: E 3,480,000, m 950,000,
    930,000 degree-1 VNs), n = 10^6, SNR 0.076, N = 150 (R15), 64-lane groups: one sampled
    lane replayed by the oracle bit-exactly; classes (2,1), (3,1), (8,0), (9,0) all run
    the specialised kernels."""
    code = make_met_code("r0.05", 10 ** 6)
    h = B.Code(code)
    assert (h.info.edges, h.info.iter_edges, h.info.m) == (3480000, 2550000, 950000)
    nf = 64
    fr = gen_batch(code, 0.076, 0, range(nf))
    dec = B.Decoder(h, nf, rule=B.RULE_EXACT, max_iter=150)
    llr_d = dec.llr_from_md(torch.from_numpy(fr["v"]).cuda(), torch.from_numpy(fr["xnorm"]).cuda(), 0.076)
    bits, iters, conv = dec.decode(llr_d, torch.from_numpy(fr["synd"].view(np.int32)).cuda())
    bits = bits.cpu().numpy().view(np.uint32)
    iters = iters.cpu().numpy()
    conv = conv.cpu().numpy()
    i = 41
    lam = bp.llr_from_md_f32(fr["v"][i], fr["xnorm"][i], 0.076)
    o = bp.decode(code, lam, fr["synd"][i], 150, rule=B.RULE_EXACT, prec=32)
    _assert_frame_equal(code, o, bits[i], iters[i], conv[i], f"lane {i}")
    assert (iters > 0).all()


def test_c6_rate002_full_size_sampled_lane():
    """Rate-0.02 column of Table 1 (R25 stand-in: E 3,337,500, m 980,000,
    960,000 degree-1 VNs, E_it 2,377,500), n = 10^6, SNR 0.029, N = 200:
    active VNs of degree 59-60 and classes (2,1), (3,1), (5,0); one sampled lane
    replayed by the oracle bit-exactly."""
    code = make_met_code("r0.02", 10 ** 6)
    h = B.Code(code)
    assert (h.info.edges, h.info.iter_edges, h.info.m) == (3337500, 2377500, 980000)
    nf = 64
    fr = gen_batch(code, 0.029, 0, range(nf))
    dec = B.Decoder(h, nf, rule=B.RULE_EXACT, max_iter=200)
    llr_d = dec.llr_from_md(torch.from_numpy(fr["v"]).cuda(), torch.from_numpy(fr["xnorm"]).cuda(), 0.029)
    bits, iters, conv = dec.decode(llr_d, torch.from_numpy(fr["synd"].view(np.int32)).cuda())
    bits = bits.cpu().numpy().view(np.uint32)
    iters = iters.cpu().numpy()
    conv = conv.cpu().numpy()
    i = 17
    lam = bp.llr_from_md_f32(fr["v"][i], fr["xnorm"][i], 0.029)
    o = bp.decode(code, lam, fr["synd"][i], 200, rule=B.RULE_EXACT, prec=32)
    _assert_frame_equal(code, o, bits[i], iters[i], conv[i], f"lane {i}")
    assert (iters > 0).all()


@pytest.mark.parametrize("d", [8, 4, 2, 1])
def test_md_alice_llr_bit_exact(c1, d):
    """GPU MD front end (metldpc_md_alice_llr, N6) bit-identical to the oracle."""
    code, h = c1
    from synth.frames import md_bob
    rng = np.random.default_rng(30 + d)
    nb = 5
    x = rng.standard_normal((nb, code.n)).astype(np.float32)
    u = rng.integers(0, 2, (nb, code.n)).astype(np.uint8)
    y = x + rng.standard_normal((nb, code.n)).astype(np.float32) * 2.5
    alpha = np.stack([md_bob(y[i].astype(np.float64), u[i], d).reshape(-1) for i in range(nb)]).astype(np.float32)
    dec = B.Decoder(h, 8)
    got = dec.md_alice_llr(torch.from_numpy(x).cuda(), torch.from_numpy(alpha).cuda(), 0.161, d=d).cpu().numpy()
    for i in range(nb):
        ref = bp.md_alice_f32(x[i], alpha[i], 0.161, d)
        assert np.array_equal(got[i].view(np.uint32), ref.view(np.uint32)), i


def test_syndrome_kernel(c1):
    """metldpc_syndrome (Step 1) = Bob's S_B of U (synth) and = the oracle's H c of decoded words."""
    code, h = c1
    fr = _frames(code, [(0.3, 3), (0.161, 3)])
    dec = B.Decoder(h, 8)
    ub = np.stack([pack_bits(u) for u in fr["u"]])
    s = dec.syndrome(torch.from_numpy(ub.view(np.int32)).cuda()).cpu().numpy().view(np.uint32)
    assert np.array_equal(s, fr["synd"])
    llr = _llr_oracle(fr)
    _, bits, iters, conv = _gpu_decode(h, llr, fr["synd"], B.RULE_EXACT, 20)
    s2 = dec.syndrome(torch.from_numpy(bits.view(np.int32)).cuda()).cpu().numpy().view(np.uint32)
    for i in range(len(llr)):
        ref = pack_bits(bp.syndrome(code, unpack_bits(bits[i], code.n)))
        assert np.array_equal(s2[i], ref)
        assert bool(conv[i]) == np.array_equal(s2[i], fr["synd"][i])


def _hub_code(D=512):
    """VN 0 of degree D (the N3 limit, kMaxVnDeg = 512) on D checks (3,0): VN 0 + a cycle of degree-2 VNs."""
    h = np.zeros((D, D + 1), np.uint8)
    for j in range(D):
        h[j, [0, 1 + j, 1 + (j + 1) % D]] = 1
    return from_dense(h)


@pytest.mark.parametrize("rule", RULES)
def test_pair_accumulator_extremes(rule):
    """64-bit pair accumulators (N3): VN 0 sums 512 saturated messages (|sum| 2.01e9 of
    the 2^31 range) with opposite signs in lanes t and t + 32, so the low word's carry into the
    high word is maximal; L and r of both halves bit-exact against M3 every iteration."""
    code = _hub_code()
    hd = B.Code(code)
    rng = np.random.default_rng(64)
    n = code.n
    llr = rng.normal(0.0, 3.0, (64, n)).astype(np.float32)
    llr[:16, 1:] = 60.0                       # lanes 0-15: every check sends VN 0 about +30
    llr[32:48, 1:] = 60.0
    llr[32:48, 1::2] = -60.0                  # lanes 32-47: alternating partner signs -> about -30
    llr[:16, 0] = 5.0
    llr[32:48, 0] = -5.0
    llr[16:32:2, 1:] = -60.0                  # lanes 16, 18, ...: negative partners
    synd = np.zeros((64, (code.m + 31) // 32), np.uint32)
    synd[48:] = np.stack([pack_bits(rng.integers(0, 2, code.m)) for _ in range(16)])
    lanes = (0, 7, 15, 16, 17, 32, 39, 47, 48, 63)
    N = 3
    traces = {i: bp.decode(code, llr[i], synd[i], N, early_term=False, rule=rule, prec=32, trace=True) for i in lanes}
    dec = B.Decoder(hd, 64, rule=rule, max_iter=N, early_term=False)
    L_t = torch.from_numpy(llr).cuda()
    S_t = torch.from_numpy(synd.view(np.int32)).cuda()
    for l in range(1, N + 1):
        dec.decode(L_t, S_t, max_iter=l)
        for i in lanes:
            r, L = dec.dump(i)
            assert np.array_equal(r.view(np.uint32), traces[i]["r_trace"][l - 1].view(np.uint32)), (l, i)
            assert np.array_equal(L.view(np.uint32), traces[i]["L_trace"][l - 1].view(np.uint32)), (l, i)
    assert abs(traces[0]["L_trace"][0][0]) > 15000 and abs(traces[32]["L_trace"][0][0]) > 15000
