"""GPU parity of the 16-bit message storage option (config msg_bits = 16, R28 / N7).

* bits, iteration counts and converged flags bit-exact against the oracle's replay M3-msg16
  (C1, both rules, frames converging at many different iterations), in group mode and with
  lane refill (the streaming decode's fresh lanes read r^0 = 0 from 16-bit rows);
* every stored message and posterior bit-exact against M3-msg16 every iteration (C1, ET off);
* teacher-forced tolerance against the plain fp64 definition M2 (north_star: |dLLR| <= 1e-3
  max(1, |LLR|) after each iteration), C1 and C2, both rules -- the storage rounding (<= 2^-11)
  is inside it;
* the pipelined / tiled / generic kernel classes (alist code with degree-17 and multi-degree-1
  checks), the no-skip layout, and a sampled C3 lane at full size.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import bp  # noqa: E402
from paper_1711_01783_b200 import binding as B  # noqa: E402
from synth.codes import make_met_code  # noqa: E402
from synth.frames import gen_batch, unpack_bits  # noqa: E402

RULES = [B.RULE_EXACT, B.RULE_PHI_LUT]
TOL = 1e-3


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1711_01783_b200.build import build
    build()


@pytest.fixture(scope="module")
def c1():
    code = make_met_code("r0.1", 2048)
    return code, B.Code(code)


def _mixed(code, parts, key):
    out = [gen_batch(code, s, key, range(i * 10000, i * 10000 + k)) | {"snr": np.full(k, s, np.float32)}
           for i, (s, k) in enumerate(parts)]
    return {k: np.concatenate([p[k] for p in out]) for k in ("u", "v", "xnorm", "synd", "snr")}


def _llr(fr):
    return np.stack([bp.llr_from_md_f32(fr["v"][i], fr["xnorm"][i], fr["snr"][i]) for i in range(len(fr["v"]))])


def _decode(h, llr, synd, rule, N, **kw):
    dec = B.Decoder(h, llr.shape[0], rule=rule, max_iter=N, msg_bits=16, **kw)
    bits, it, cv = dec.decode(torch.from_numpy(llr).cuda(), torch.from_numpy(synd.view(np.int32)).cuda())
    torch.cuda.synchronize()
    return dec, bits.cpu().numpy().view(np.uint32), it.cpu().numpy(), cv.cpu().numpy()


def _check(code, llr, synd, N, rule, bits_row, it, cv, tag, no_skip=False):
    o = bp.decode(code, llr, synd, N, rule=rule, prec=32, msg16=True, no_skip=no_skip)
    assert it == o["iters"], (tag, it, o["iters"])
    assert bool(cv) == o["converged"], tag
    assert np.array_equal(unpack_bits(bits_row, code.n), o["bits"]), tag
    return o


@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("refill", [False, True])
def test_c1_msg16_bits_iters_flags(c1, rule, refill):
    code, h = c1
    fr = _mixed(code, [(0.161, 20), (0.2, 30), (0.3, 30), (0.5, 20)], key=70)
    llr = _llr(fr)
    _, bits, it, cv = _decode(h, llr, fr["synd"], rule, 100, lane_refill=refill)
    nconv = 0
    for i in range(len(llr)):
        nconv += _check(code, llr[i], fr["synd"][i], 100, rule, bits[i], it[i], cv[i], f"frame {i}")["converged"]
    assert 20 <= nconv < len(llr)


@pytest.mark.parametrize("rule", RULES)
def test_c1_msg16_messages_every_iteration(c1, rule):
    code, h = c1
    fr = _mixed(code, [(0.161, 18), (0.3, 18)], key=71)
    llr = _llr(fr)
    lanes = (0, 1, 17, 18, 32, 33, 34, 35)   # both halves of the pair words (N3, N7)
    N = 30
    traces = {i: bp.decode(code, llr[i], fr["synd"][i], N, early_term=False, rule=rule, prec=32, trace=True, msg16=True)
              for i in lanes}
    dec = B.Decoder(h, len(llr), rule=rule, max_iter=N, early_term=False, msg_bits=16)
    L_t, S_t = torch.from_numpy(llr).cuda(), torch.from_numpy(fr["synd"].view(np.int32)).cuda()
    for l in range(1, N + 1):
        dec.decode(L_t, S_t, max_iter=l)
        for i in lanes:
            r, L = dec.dump(i)
            assert np.array_equal(r.view(np.uint32), traces[i]["r_trace"][l - 1].view(np.uint32)), (l, i)
            assert np.array_equal(L.view(np.uint32), traces[i]["L_trace"][l - 1].view(np.uint32)), (l, i)


def _teacher_forced(code, h, rule, fr, llr, N, lanes):
    dec = B.Decoder(h, len(llr), rule=rule, max_iter=N, early_term=False, lane_refill=False, msg_bits=16)
    L_t, S_t = torch.from_numpy(llr).cuda(), torch.from_numpy(fr["synd"].view(np.int32)).cuda()
    E_it = h.info.iter_edges
    act = np.flatnonzero(np.diff(code.vn_ptr) >= 2)
    prev = {i: (np.zeros(E_it), llr[i][act].astype(np.float64)) for i in lanes}
    worst = 0.0
    dec.decode(L_t, S_t, max_iter=1)
    for l in range(1, N + 1):
        if l > 1:
            dec.step(1)
        for i in lanes:
            r, L = dec.dump(i)
            r_ref, L_ref = bp.step64(code, llr[i].astype(np.float64), fr["synd"][i], prev[i][0], prev[i][1], rule=rule)
            for got, ref, what in ((r, r_ref, "r"), (L, L_ref, "L")):
                err = np.abs(got.astype(np.float64) - ref) / np.maximum(1.0, np.abs(ref))
                worst = max(worst, float(err.max()))
                assert err.max() <= TOL, (what, l, i, float(err.max()))
            prev[i] = (r.astype(np.float64), L.astype(np.float64))
    return worst


@pytest.mark.parametrize("rule", RULES)
def test_msg16_teacher_forced_c1(c1, rule):
    code, h = c1
    fr = _mixed(code, [(0.161, 2), (0.3, 2)], key=72)
    worst = _teacher_forced(code, h, rule, fr, _llr(fr), 30, range(4))
    assert 1e-4 < worst < TOL   # the storage rounding shows, and stays inside the tolerance


@pytest.mark.parametrize("rule", RULES)
def test_msg16_teacher_forced_c2(rule):
    code = make_met_code("r0.1", 65536)
    h = B.Code(code)
    fr = _mixed(code, [(0.161, 40), (0.2, 24)], key=73)
    _teacher_forced(code, h, rule, fr, _llr(fr), 10, (5, 60))


def test_msg16_generic_classes_and_no_skip():
    """Kernel classes beyond the pipelined ones: random codes covering every CN-degree window
    (0-4, 5-8, 9-12, 13-16, 17-32: pipelined, tiled and generic kernels, several degree-1 slots
    per check), plus the no-skip layout (every inner check a (4,0) class)."""
    from synth.codes import random_code
    from synth.frames import pack_bits
    rng = np.random.default_rng(74)
    for t, (n, m, deg) in enumerate([(60, 20, (2, 3)), (80, 12, (2, 4)), (120, 12, (2, 3)), (90, 16, (2, 3))]):
        for _ in range(100):
            code = random_code(n, m, rng, frac_deg1=0.3, act_deg=deg)
            if code.cn_degree.max() <= 32:
                break
        h = B.Code(code)
        u = rng.integers(0, 2, n).astype(np.uint8)
        s = (code.dense().astype(int) @ u) % 2
        llr = ((1 - 2.0 * u) * rng.uniform(0.2, 2.5, (8, n))).astype(np.float32)
        llr[:, :5] *= -1
        synd = np.stack([pack_bits(s)] * 8)
        for rule in RULES:
            _, bits, it, cv = _decode(h, llr, synd, rule, 30, lane_refill=False)
            for i in range(8):
                _check(code, llr[i], synd[i], 30, rule, bits[i], it[i], cv[i], f"code {t} frame {i}")
    c1 = make_met_code("r0.1", 2048)
    hn = B.Code(c1, no_skip=True)
    fr = _mixed(c1, [(0.2, 8), (0.4, 8)], key=76)
    llr = _llr(fr)
    _, bits, it, cv = _decode(hn, llr, fr["synd"], B.RULE_EXACT, 80)
    for i in range(len(llr)):
        _check(c1, llr[i], fr["synd"][i], 80, B.RULE_EXACT, bits[i], it[i], cv[i], f"no-skip {i}", no_skip=True)


def test_msg16_c3_full_size_sampled():
    """C3 (n = 10^6) at SNR 0.19 with lane refill: 128 frames, three sampled frames (converged
    and failed) bit-exact against M3-msg16."""
    code = make_met_code("r0.1", 10 ** 6)
    h = B.Code(code)
    snr, nf = 0.19, 128
    fr = gen_batch(code, snr, 77, range(nf))
    dec = B.Decoder(h, nf, max_iter=100, lane_refill=True, msg_bits=16)
    llr = dec.llr_from_md(torch.from_numpy(fr["v"]).cuda(), torch.from_numpy(fr["xnorm"]).cuda(), snr)
    bits, it, cv = dec.decode(llr, torch.from_numpy(fr["synd"].view(np.int32)).cuda())
    torch.cuda.synchronize()
    bits, it, cv = bits.cpu().numpy().view(np.uint32), it.cpu().numpy(), cv.cpu().numpy()
    assert 0 < cv.sum() < nf
    sample = [int(np.flatnonzero(cv == 0)[0]), int(np.flatnonzero(cv == 1)[0]),
              int(np.argmax(np.where(cv == 1, it, -1)))]

    def one(i):
        lam = bp.llr_from_md_f32(fr["v"][i], fr["xnorm"][i], snr)
        return bp.decode(code, lam, fr["synd"][i], 100, prec=32, msg16=True)

    with ThreadPoolExecutor(len(sample)) as ex:
        res = list(ex.map(one, sample))
    for i, o in zip(sample, res):
        assert it[i] == o["iters"] and bool(cv[i]) == o["converged"], (i, it[i], o["iters"])
        assert np.array_equal(unpack_bits(bits[i], code.n), o["bits"]), i


def test_msg16_config_validation(c1):
    code, h = c1
    with pytest.raises(B.MetLdpcError):
        B.Decoder(h, 8, msg_bits=16, lanes_per_group=32)
    with pytest.raises(B.MetLdpcError):
        B.Decoder(h, 8, msg_bits=8)
