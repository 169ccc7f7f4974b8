"""GPU parity of the paths the bench runs, against the CPU oracle.

* metldpc_decode_md_host (the API behind bench's `e2e`): streaming (lane refill) and group
  mode, d = 8/4/2/1 with and without |x|, a batch larger than the streaming host path's
  staging (two super-chunks), against the device path and oracle M3.
* C3 at full size (n = 10^6) at a converging SNR with lane refill: partial refill waves mix
  fresh and iterating lanes; sampled converged and failed lanes against M3.
* Teacher-forced tolerance against the plain definition M2 (north_star: |dLLR| <=
  1e-3 max(1, |LLR|) after each iteration): the GPU state at l - 1 (metldpc_debug_dump) is
  stepped once by M2 (fp64) and by the GPU (metldpc_debug_step), for C1 and C2, both rules.
* metldpc_batch_counters against numpy sums, invalid frames included.
Inputs are seeded synthetic frames from synth/ (never from the CUDA path).
"""
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import bp  # noqa: E402
from paper_1711_01783_b200 import binding as B  # noqa: E402
from synth.codes import make_met_code  # noqa: E402
from synth.frames import gen_batch, unpack_bits  # noqa: E402

RULES = [B.RULE_EXACT, B.RULE_PHI_LUT]
TOL = 1e-3   # BASELINE north_star: |dLLR| <= 1e-3 max(1, |LLR|)


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


def _mixed(code, parts, key, d=8):
    """Frames at several SNRs: [(snr, count)] -> dict with per-frame snr."""
    out = [gen_batch(code, s, key, range(i * 10000, i * 10000 + k), d=d) | {"snr": np.full(k, s, np.float32)}
           for i, (s, k) in enumerate(parts)]
    return {k: np.concatenate([p[k] for p in out]) for k in ("u", "v", "xnorm", "synd", "snr")}


def _check_frame(code, llr, synd, N, rule, bits_row, it, cv, tag):
    o = bp.decode(code, llr, synd, N, early_term=True, rule=rule, prec=32)
    assert it == o["iters"], (tag, it, o["iters"])
    assert bool(cv) == o["converged"], tag
    assert np.array_equal(unpack_bits(bits_row, code.n), o["bits"]), tag
    return o


# ----------------------------------------------------------------------------- decode_md_host

@pytest.mark.parametrize("d,with_norm", [(8, True), (8, False), (4, True), (2, True), (1, True)])
@pytest.mark.parametrize("refill,groups", [(True, 1), (True, 2), (False, 1), (False, 2)])
def test_decode_md_host_parity(c1, d, with_norm, refill, groups):
    """metldpc_decode_md_host (H2D, LLR, decode, D2H inside the call) == the device path
    (metldpc_llr_from_md + metldpc_decode) bit for bit, and sampled frames == M3; a ragged
    batch of 150 frames at SNR 0.2 (the host call takes one snr), where frames latch at many
    different iterations and some fail."""
    code, h = c1
    snr = 0.2
    fr = _mixed(code, [(snr, 150)], key=40 + d, d=d)
    nb = len(fr["v"])
    v = np.ascontiguousarray(fr["v"])
    xn = np.ascontiguousarray(fr["xnorm"]) if with_norm else None
    sy = np.ascontiguousarray(fr["synd"])
    dec = B.Decoder(h, nb, rule=B.RULE_EXACT, max_iter=60, groups_in_flight=groups, lane_refill=refill)
    hb, hi, hc = dec.decode_md_host(torch.from_numpy(v).pin_memory(),
                                    torch.from_numpy(xn).pin_memory() if xn is not None else None,
                                    torch.from_numpy(sy.view(np.int32)).pin_memory(), snr, d=d)
    hb, hi, hc = (np.asarray(x) for x in (hb, hi, hc))
    # device path
    vt = torch.from_numpy(v).cuda()
    llr = dec.llr_from_md(vt, torch.from_numpy(xn).cuda() if xn is not None else None, snr, d=d)
    db, di, dc = dec.decode(llr, torch.from_numpy(sy.view(np.int32)).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(hb.view(np.uint32), db.cpu().numpy().view(np.uint32))
    assert np.array_equal(hi, di.cpu().numpy()) and np.array_equal(hc, dc.cpu().numpy())
    assert 0 < hc.sum() < nb or d != 8
    for i in (0, 37, 77, nb - 1):
        lam = bp.llr_from_md_f32(v[i], xn[i] if xn is not None else None, snr, d)
        _check_frame(code, lam, sy[i], 60, B.RULE_EXACT, hb.view(np.uint32)[i], hi[i], hc[i], f"d{d} frame {i}")


def test_decode_host_streaming_superchunks(c1):
    """A batch larger than the streaming host path's staging (2048 frames): two super-chunks,
    each fed in 32-frame chunks to the running decode; == group mode and == M3 (sampled)."""
    code, h = c1
    fr = _mixed(code, [(0.18, 700), (0.25, 700), (0.5, 700)], key=77)
    llr = np.stack([bp.llr_from_md_f32(fr["v"][i], fr["xnorm"][i], fr["snr"][i]) for i in range(len(fr["v"]))])
    llr[1000, 5] = np.inf
    nb = len(llr)
    sy = np.ascontiguousarray(fr["synd"])
    out = {}
    for refill in (True, False):
        dec = B.Decoder(h, nb, rule=B.RULE_PHI_LUT, max_iter=40, lane_refill=refill, groups_in_flight=2)
        out[refill] = tuple(np.asarray(x) for x in dec.decode_host(llr, sy))
        dec.close()
    for a, b in zip(out[True], out[False]):
        assert np.array_equal(a, b)
    bits, iters, conv = out[True]
    assert iters[1000] == -1 and conv[1000] == 0
    assert len(set(iters.tolist())) > 8
    for i in (0, 699, 1400, 2047, 2048, 2099):
        _check_frame(code, llr[i], sy[i], 40, B.RULE_PHI_LUT, bits.view(np.uint32)[i], iters[i], conv[i], f"frame {i}")


# ----------------------------------------------------------------------------- C3 with lane refill

def test_c3_full_size_refill_converging():
    """C3 code at full size (n = 10^6, rate 0.1, N = 100) at SNR 0.19, where most frames
    converge: 192 frames (96 distinct, tiled, so identical frames sit in different lanes and
    refill waves) through the streaming decode (lane refill, 64-lane groups, the bench's launch
    configuration); six sampled frames, converged and failed, replayed by M3 bit-exactly, and
    every tiled copy of a frame decoded identically."""
    code = make_met_code("r0.1", 10 ** 6)
    h = B.Code(code)
    snr, nd, nf = 0.19, 96, 192
    from multiprocessing import get_context
    with get_context("fork").Pool(8) as pool:
        frs = pool.starmap(_gen_c3, [(snr, f) for f in range(nd)])
    v = np.stack([f[0] for f in frs])
    xn = np.stack([f[1] for f in frs])
    sy = np.stack([f[2] for f in frs])
    idx = np.concatenate([np.arange(nd), np.arange(nd)[::-1]])          # copies in other lanes
    dec = B.Decoder(h, nf, rule=B.RULE_EXACT, max_iter=100, lane_refill=True)
    llr = dec.llr_from_md(torch.from_numpy(v[idx]).cuda(), torch.from_numpy(xn[idx]).cuda(), snr)
    bits, iters, conv = dec.decode(llr, torch.from_numpy(sy[idx].view(np.int32)).cuda())
    torch.cuda.synchronize()
    bits, iters, conv = bits.cpu().numpy().view(np.uint32), iters.cpu().numpy(), conv.cpu().numpy()
    # copies agree
    for j in range(nd):
        k = nf - 1 - j
        assert np.array_equal(bits[j], bits[k]) and iters[j] == iters[k] and conv[j] == conv[k], j
    assert 0 < conv.sum() < nf and len(set(iters.tolist())) > 10
    # sampled frames: some converged, some failed
    failed = [int(i) for i in np.flatnonzero(conv[:nd] == 0)[:2]]
    good = [int(i) for i in np.flatnonzero(conv[:nd] == 1)]
    good = [good[0], good[len(good) // 2], good[-1], int(np.argmax(np.where(conv[:nd] == 1, iters[:nd], -1)))]
    sample = failed + good
    assert len(failed) >= 1 and len(sample) >= 4

    def one(i):
        lam = bp.llr_from_md_f32(v[i], xn[i], snr)
        return bp.decode(code, lam, sy[i], 100, early_term=True, rule=B.RULE_EXACT, prec=32)

    with ThreadPoolExecutor(len(sample)) as ex:
        res = list(ex.map(one, sample))
    for i, o in zip(sample, res):
        assert iters[i] == o["iters"] and bool(conv[i]) == o["converged"], (i, iters[i], o["iters"])
        assert np.array_equal(unpack_bits(bits[i], code.n), o["bits"]), i


def _gen_c3(snr, f):
    from synth.frames import gen_frame
    code = make_met_code("r0.1", 10 ** 6)
    fr = gen_frame(code, snr, 3, f)
    return fr["v"], fr["xnorm"], fr["synd"]


# ----------------------------------------------------------------------------- teacher-forced vs M2

def _teacher_forced(code, h, rule, fr, llr, N, lanes):
    dec = B.Decoder(h, len(llr), rule=rule, max_iter=N, early_term=False, lane_refill=False)
    L_t = torch.from_numpy(llr).cuda()
    S_t = torch.from_numpy(fr["synd"].view(np.int32)).cuda()
    E_it, n_a = h.info.iter_edges, h.info.n_active
    act = np.flatnonzero(np.diff(code.vn_ptr) >= 2)
    prev = {i: (np.zeros(E_it), llr[i][act].astype(np.float64)) for i in lanes}   # l = 0: r = 0, L = lambda
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
                assert err.max() <= TOL, (what, l, i, float(err.max()), int(err.argmax()))
            prev[i] = (r.astype(np.float64), L.astype(np.float64))
    return worst


@pytest.mark.parametrize("rule", RULES)
def test_teacher_forced_tolerance_c1(c1, rule):
    """C1: 30 iterations, 4 lanes (SNR 0.161 and 0.3), every edge message and posterior."""
    code, h = c1
    fr = _mixed(code, [(0.161, 2), (0.3, 2)], key=60)
    llr = np.stack([bp.llr_from_md_f32(fr["v"][i], fr["xnorm"][i], fr["snr"][i]) for i in range(4)])
    worst = _teacher_forced(code, h, rule, fr, llr, 30, range(4))
    assert worst < TOL


@pytest.mark.parametrize("rule", RULES)
def test_teacher_forced_tolerance_c2(rule):
    """C2 (n = 65,536, 64-lane batch): 12 iterations on two sampled lanes of the batch."""
    code = make_met_code("r0.1", 65536)
    h = B.Code(code)
    fr = _mixed(code, [(0.161, 40), (0.2, 24)], key=61)
    llr = np.stack([bp.llr_from_md_f32(fr["v"][i], fr["xnorm"][i], fr["snr"][i]) for i in range(64)])
    _teacher_forced(code, h, rule, fr, llr, 12, (3, 50))


def test_debug_step_matches_decode(c1):
    """decode(N = l) == decode(N = 1) + debug_step(l - 1), message for message (M3 traces
    then pin both), and debug_step refuses to run after a streaming decode."""
    code, h = c1
    fr = _mixed(code, [(0.2, 3)], key=62)
    llr = np.stack([bp.llr_from_md_f32(fr["v"][i], fr["xnorm"][i], fr["snr"][i]) for i in range(3)])
    L_t, S_t = torch.from_numpy(llr).cuda(), torch.from_numpy(fr["synd"].view(np.int32)).cuda()
    dec = B.Decoder(h, 3, max_iter=20, early_term=False)
    dec.decode(L_t, S_t, max_iter=1)
    dec.step(6)
    o = bp.decode(code, llr[1], fr["synd"][1], 7, early_term=False, prec=32, trace=True)
    r, L = dec.dump(1)
    assert np.array_equal(r.view(np.uint32), o["r_trace"][-1].view(np.uint32))
    assert np.array_equal(L.view(np.uint32), o["L_trace"][-1].view(np.uint32))
    dec2 = B.Decoder(h, 3, max_iter=20, early_term=True, lane_refill=True)
    dec2.decode(L_t, S_t)
    with pytest.raises(B.MetLdpcError):
        dec2.step(1)


# ----------------------------------------------------------------------------- counters (a7)

def test_batch_counters(c1):
    """metldpc_batch_counters adds {frames, converged, sum of iterations over valid frames,
    invalid frames} into its output; checked against numpy on real decode results with
    invalid frames, and on a large synthetic batch (several blocks, atomics)."""
    code, h = c1
    fr = _mixed(code, [(0.2, 40), (0.5, 30)], key=63)
    llr = np.stack([bp.llr_from_md_f32(fr["v"][i], fr["xnorm"][i], fr["snr"][i]) for i in range(70)])
    llr[[3, 44], 9] = np.nan
    dec = B.Decoder(h, 70, max_iter=50)
    _, it, cv = dec.decode(torch.from_numpy(llr).cuda(), torch.from_numpy(fr["synd"].view(np.int32)).cuda())
    out = torch.zeros(4, dtype=torch.int64, device="cuda")
    dec.counters(it, cv, out)
    dec.counters(it, cv, out)          # accumulates
    torch.cuda.synchronize()
    itn, cvn = it.cpu().numpy(), cv.cpu().numpy()
    ref = np.array([70, cvn.sum(), itn[itn >= 0].sum(), (itn < 0).sum()], np.int64)
    assert ref[3] == 2 and 0 < ref[1] < 70
    assert out.cpu().numpy().tolist() == (2 * ref).tolist()
    rng = np.random.default_rng(5)
    big = 100_003
    it2 = rng.integers(-1, 150, big).astype(np.int32)
    cv2 = (rng.random(big) < 0.3).astype(np.uint8)
    dec2 = B.Decoder(h, 8)
    out2 = torch.zeros(4, dtype=torch.int64, device="cuda")
    B.metldpc_batch_counters(dec2.h, big, torch.from_numpy(it2).cuda(), torch.from_numpy(cv2).cuda(), out2)
    torch.cuda.synchronize()
    assert out2.cpu().numpy().tolist() == [big, int(cv2.sum()), int(it2[it2 >= 0].sum()), int((it2 < 0).sum())]


# ----------------------------------------------------------------------------- headline config

def test_r01de_c1_bits_iters_flags(c1):
    """The density-evolution stand-in (r0.1de, R29) at C1 size: its kernel classes
    (inner (2,1) and (3,1) checks in the ring kernel, core (13,0)/(14,0) checks in the tiled
    kernel) bit-exact against M3 on BIAWGN frames (R31), both message formats."""
    from synth.frames import gen_batch_biawgn
    code = make_met_code("r0.1de", 2048)
    h = B.Code(code)
    fr = [gen_batch_biawgn(code, s, 80, range(i * 100, i * 100 + 16)) for i, s in enumerate((0.2, 0.35, 0.6))]
    llr = np.concatenate([f["llr"] for f in fr])
    sy = np.concatenate([f["synd"] for f in fr])
    for msg in (32, 16):
        dec = B.Decoder(h, len(llr), max_iter=100, msg_bits=msg)
        bits, it, cv = dec.decode(torch.from_numpy(llr).cuda(), torch.from_numpy(sy.view(np.int32)).cuda())
        torch.cuda.synchronize()
        bits, it, cv = bits.cpu().numpy().view(np.uint32), it.cpu().numpy(), cv.cpu().numpy()
        nconv = 0
        for i in range(len(llr)):
            o = bp.decode(code, llr[i], sy[i], 100, prec=32, msg16=msg == 16)
            assert it[i] == o["iters"] and bool(cv[i]) == o["converged"], (msg, i)
            assert np.array_equal(unpack_bits(bits[i], code.n), o["bits"]), (msg, i)
            nconv += o["converged"]
        assert 0 < nconv < len(llr)


def _gen_c3_biawgn(snr, f):
    from synth.frames import gen_frame_biawgn
    code = make_met_code("r0.1de", 10 ** 6)
    fr = gen_frame_biawgn(code, snr, 81, f)
    return fr["llr"], fr["synd"], fr["u"]


def test_headline_config_sampled_frames():
    """The bench's headline configuration (r0.1de, n = 10^6, BIAWGN input at SNR 0.161, N = 100,
    early termination + lane refill, 64-lane groups, fp32 messages): 128 frames (64 distinct, each
    twice in different lanes / refill waves); three sampled frames bit-exact against M3, every
    copy decoded identically, and the decoder converges there (FER < 0.5, mean iterations < 100)."""
    code = make_met_code("r0.1de", 10 ** 6)
    h = B.Code(code)
    snr, nd = 0.161, 64
    from multiprocessing import get_context
    with get_context("fork").Pool(8) as pool:
        frs = pool.starmap(_gen_c3_biawgn, [(snr, f) for f in range(nd)])
    llr = np.stack([f[0] for f in frs])
    sy = np.stack([f[1] for f in frs])
    idx = np.concatenate([np.arange(nd), np.arange(nd)[::-1]])
    dec = B.Decoder(h, 2 * nd, max_iter=100, lane_refill=True)
    bits, it, cv = dec.decode(torch.from_numpy(llr[idx]).cuda(), torch.from_numpy(sy[idx].view(np.int32)).cuda())
    torch.cuda.synchronize()
    bits, it, cv = bits.cpu().numpy().view(np.uint32), it.cpu().numpy(), cv.cpu().numpy()
    for j in range(nd):
        k = 2 * nd - 1 - j
        assert np.array_equal(bits[j], bits[k]) and it[j] == it[k] and cv[j] == cv[k], j
    assert cv.mean() > 0.5 and it.mean() < 100
    good = [int(i) for i in np.flatnonzero(cv[:nd] == 1)]
    sample = [good[0], int(np.argmax(np.where(cv[:nd] == 1, it[:nd], -1)))]
    bad = np.flatnonzero(cv[:nd] == 0)
    if bad.size:
        sample.append(int(bad[0]))

    def one(i):
        return bp.decode(code, llr[i], sy[i], 100, prec=32)

    with ThreadPoolExecutor(len(sample)) as ex:
        res = list(ex.map(one, sample))
    for i, o in zip(sample, res):
        assert it[i] == o["iters"] and bool(cv[i]) == o["converged"], (i, it[i], o["iters"])
        assert np.array_equal(unpack_bits(bits[i], code.n), o["bits"]), i


# ----------------------------------------------------------------------------- A/B kernel alternatives

_ALT_SCRIPT = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
from oracle import bp
from paper_1711_01783_b200 import binding as B
from synth.codes import make_met_code, random_code
from synth.frames import gen_batch, unpack_bits
for code in (make_met_code("r0.1", 2048), random_code(600, 240, np.random.default_rng(11), frac_deg1=0.3, act_deg=(2, 5))):
    h = B.Code(code)
    fr = gen_batch(code, 0.3, 5, range(40))
    llr = np.stack([bp.llr_from_md_f32(fr["v"][i], fr["xnorm"][i], 0.3) for i in range(40)])
    for rule in (B.RULE_EXACT, B.RULE_PHI_LUT):
        for msg in (32, 16):
            dec = B.Decoder(h, 40, rule=rule, max_iter=30, msg_bits=msg)
            bits, it, cv = dec.decode(torch.from_numpy(llr).cuda(), torch.from_numpy(fr["synd"].view(np.int32)).cuda())
            torch.cuda.synchronize()
            bits = bits.cpu().numpy().view(np.uint32)
            for i in (0, 7, 33, 39):
                o = bp.decode(code, llr[i], fr["synd"][i], 30, rule=rule, prec=32, msg16=(msg == 16))
                assert it[i].item() == o["iters"] and bool(cv[i].item()) == o["converged"], (code.name, rule, msg, i)
                assert np.array_equal(unpack_bits(bits[i], code.n), o["bits"]), (code.name, rule, msg, i)
print("ok")
"""


@pytest.mark.parametrize("env", ["METLDPC_RING=0", "METLDPC_RING_CORE=0", "METLDPC_PIPE=0"])
def test_alternative_kernel_paths(env):
    """The A/B alternatives kept in the library (per-warp pipeline k_cn_pipe, register-only k_cn_tile
    for the core or for all exact classes) decode bit-exactly like M3: a subprocess per switch, since
    the switches are read once per process."""
    import os
    import subprocess
    import sys
    root = str(Path(__file__).resolve().parents[1])
    k, v = env.split("=")
    r = subprocess.run([sys.executable, "-c", _ALT_SCRIPT, root], env=dict(os.environ, **{k: v}),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("msg_bits", [32, 16])
def test_idle_lanes_over_reused_memory(msg_bits):
    """Lanes that never hold a frame (40 frames in a 64-lane streaming group) are computed too; the
    decoder clears their degree-1 priors at allocation, so memory left by earlier, destroyed decoders
    cannot push the checks' unclamped output phi lookups out of the table (this sequence of codes and
    decoders created and destroyed faulted before the clear)."""
    code = make_met_code("r0.1", 2048)
    fr = gen_batch(code, 0.3, 5, range(40))
    llr = np.stack([bp.llr_from_md_f32(fr["v"][i], fr["xnorm"][i], 0.3) for i in range(40)])
    refs = {i: bp.decode(code, llr[i], fr["synd"][i], 30, prec=32, msg16=(msg_bits == 16)) for i in (0, 13, 39)}
    L_t, S_t = torch.from_numpy(llr).cuda(), torch.from_numpy(fr["synd"].view(np.int32)).cuda()
    h = dec = None
    for rep in range(6):   # each code / decoder is created before its predecessor is destroyed
        h = B.Code(code)
        for rule in (B.RULE_EXACT, B.RULE_PHI_LUT):
            dec = B.Decoder(h, 40, rule=rule, max_iter=30, msg_bits=msg_bits, lane_refill=True)
            bits, it, cv = dec.decode(L_t, S_t)
            torch.cuda.synchronize()
            if rule == B.RULE_EXACT:
                bits = bits.cpu().numpy().view(np.uint32)
                for i, o in refs.items():
                    assert it[i].item() == o["iters"] and np.array_equal(unpack_bits(bits[i], code.n), o["bits"]), (rep, i)
