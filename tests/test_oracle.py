"""CPU pins of the oracle (oracle/) against what the paper and the mathematics fix.

Nothing here touches the CUDA path.  Each test names the passage it pins.
"""
import json
import math

import numpy as np
import pytest

from oracle import bp, brute, literal
from synth.codes import from_dense, random_code, tree_code
from synth.frames import gen_frame, pack_bits

GOLD = json.loads((__import__("pathlib").Path(__file__).parent / "golden" / "spec_examples.json").read_text())


def llr_of_ratio(q):
    """Eq. (1) ratio q = P(1)/P(0)  ->  lambda = ln P(0)/P(1) = -ln q."""
    return -math.log(q)


# ----------------------------------------------------------------- phi

def test_phi_involution_and_closed_form():
    # phi(phi(y)) = y and phi(y) = -ln tanh(y/2): an independent closed form.
    for y in np.geomspace(1e-6, 30, 200):
        assert abs(bp.phi_def(bp.phi_def(y)) - y) <= 1e-9 * max(1.0, y)
        assert abs(bp.phi_def(y) - (-math.log(math.tanh(y / 2)))) <= 1e-12 * max(1.0, bp.phi_def(y))
    assert math.isinf(bp.phi_def(0.0))


@pytest.mark.parametrize("rule,abs_tol,tail_rel", [(bp.RULE_EXACT, 2.5e-6, 3e-3), (bp.RULE_PHI_LUT, 1.5e-4, 4e-2)])
def test_phi32_table_error_bound(rule, abs_tol, tail_rel):
    """DESIGN.md N2: the fp32 tables against the definition over [2^-44, 64)."""
    rng = np.random.default_rng(0)
    ys = np.exp(rng.uniform(math.log(2.0 ** -44), math.log(63.9), 4000)).astype(np.float32)
    for y in ys:
        ref = bp.phi_def(float(y))
        got = bp.phi32(rule, float(y))
        if ref < 30:
            assert abs(got - ref) <= abs_tol + 2e-7 * ref, (y, got, ref)
        if y < 32:
            assert abs(got - ref) <= tail_rel * ref + 2e-7 * ref + 1e-30, (y, got, ref)
    # out-of-range conventions: below 2^-44 -> phi(2^-44) (> R_MAX, so it clamps); >= 64 -> 0
    assert bp.phi32(rule, 0.0) > 30.0
    assert bp.phi32(rule, 64.0) == 0.0
    assert bp.phi32(rule, 1e30) == 0.0


def test_phi64_lut_hits_knots():
    # PHI_LUT in fp64 interpolates linearly between exact knot values (reading R5).
    for e in (-10, -1, 0, 3):
        for j in (0, 7, 31):
            y = math.ldexp(1 + j / 32, e)
            assert bp.phi64(bp.RULE_PHI_LUT, y) == pytest.approx(bp.phi_def(y), rel=1e-15)


# ----------------------------------------------------------------- SPEC worked examples

@pytest.mark.parametrize("ex", GOLD["cn_update"], ids=lambda e: e["cite"])
@pytest.mark.parametrize("prec", [32, 64])
def test_cn_update_spec(ex, prec):
    """Eqs. (2)-(3): one CN, target VN of degree 1 with lambda = 0
    so its posterior after one iteration IS the CN message."""
    others = ex["other_ratios"]
    d = len(others) + 1
    code = from_dense(np.ones((1, d), np.uint8))
    lam = np.array([0.0] + [llr_of_ratio(q) for q in others])
    o = bp.decode(code, lam, pack_bits([ex["s"]]), 1, early_term=False, prec=64, posterior=True)
    assert o["post"][0] == pytest.approx(llr_of_ratio(ex["r"]), abs=1e-12)
    if prec == 32:   # fp32 replay (EXACT table) within the table bound
        o32 = bp.decode(code, lam, pack_bits([ex["s"]]), 1, early_term=False, prec=32)
        assert o32["bits"][0] == int(llr_of_ratio(ex["r"]) < 0)
    # the literal ratio-domain equations give the printed number directly
    o1 = literal.decode_ratio(np.ones((1, d)), lam, [ex["s"]], 1, early_term=False)
    assert math.exp(-o1["post"][0]) == pytest.approx(ex["r"], rel=1e-12)


@pytest.mark.parametrize("ex", GOLD["vn_update"], ids=lambda e: e["cite"])
def test_vn_update_spec(ex):
    """Eq. (4): q_ij = q0_i prod_{j' != j} r_j'i.  VN 0 has two
    degree-2 CNs that pass the degree-1 partners' priors through unchanged and
    a third CN C whose degree-1 partner (lambda = 0) reads q_0C at l = 2."""
    ra, rb = ex["other_r"]
    # VNs: 0 (target), 1 (partner on CN A), 2 (partner on CN B), 3 (partner on CN C)
    h = np.array([[1, 1, 0, 0], [1, 0, 1, 0], [1, 0, 0, 1]], np.uint8)
    code = from_dense(h)
    lam = np.array([llr_of_ratio(ex["q0"]), llr_of_ratio(ra), llr_of_ratio(rb), 0.0])
    o = bp.decode(code, lam, pack_bits([0, 0, 0]), 2, early_term=False, prec=64, posterior=True)
    assert math.exp(-o["post"][3]) == pytest.approx(ex["q"], rel=1e-9)
    o1 = literal.decode_ratio(h, lam, [0, 0, 0], 2, early_term=False)
    assert math.exp(-o1["post"][3]) == pytest.approx(ex["q"], rel=1e-9)


@pytest.mark.parametrize("ex", GOLD["decision"], ids=lambda e: e["cite"])
@pytest.mark.parametrize("prec", [32, 64])
def test_decision_spec(ex, prec):
    """Step 5 / Eq. (5): c = 1 iff posterior ratio > 1; tie -> 0."""
    if "q0" in ex:
        # degree-1 VN 0 with prior q0, its CN (degree 2) passes partner VN 1's prior = r
        code = from_dense(np.array([[1, 1]], np.uint8))
        lam = np.array([llr_of_ratio(ex["q0"]), llr_of_ratio(ex["r"])])
    else:
        # VN 0 on a degree-2 CN whose partner has lambda = 0 -> message 0, posterior = prior
        code = from_dense(np.array([[1, 1]], np.uint8))
        lam = np.array([llr_of_ratio(ex["posterior_ratio"]), 0.0])
    o = bp.decode(code, lam, pack_bits([0]), 1, early_term=False, prec=prec)
    assert int(o["bits"][0]) == ex["bit"]


@pytest.mark.parametrize("ex", GOLD["syndrome"], ids=lambda e: e["cite"])
def test_syndrome_spec(ex):
    code = from_dense(np.array(ex["H"], np.uint8))
    assert list(bp.syndrome(code, np.array(ex["c"], np.uint8))) == ex["s"]


@pytest.mark.parametrize("ex", GOLD["layout"], ids=lambda e: e["cite"])
def test_layout_spec(ex):
    code = from_dense(np.array(ex["H"], np.uint8))
    assert list(code.vn_degree) == ex["vn_degrees"]
    E_it, n_a = bp.graph_sizes(code)
    assert E_it == ex["iter_edges"] and n_a == ex["n_active"]


# ----------------------------------------------------------------- ground truth on tiny codes

@pytest.mark.parametrize("seed", range(12))
def test_tree_codes_equal_bitwise_map(seed):
    """BP is exact on cycle-free graphs: after >= diameter iterations the M2
    posterior equals the brute-force bitwise MAP over the coset {c: Hc = S_B}."""
    rng = np.random.default_rng(100 + seed)
    tc = tree_code(rng, n_cn=int(rng.integers(2, 6)))
    h = tc.dense()
    lam = rng.normal(0.4, 1.5, tc.n)
    s = rng.integers(0, 2, tc.m)
    ref = brute.bitwise_map(h, s, lam)
    o = bp.decode(tc, lam, pack_bits(s), 2 * tc.m + 2, early_term=False, prec=64, posterior=True)
    assert np.allclose(o["post"], ref, atol=1e-9, rtol=1e-9)
    o1 = literal.decode_ratio(h, lam, s, 2 * tc.m + 2, early_term=False)
    assert np.allclose(o1["post"], ref, atol=1e-9, rtol=1e-9)
    # fp32 replay, both rules: decisions equal the MAP decisions (|MAP LLR| bounded away from 0)
    for rule in (bp.RULE_EXACT, bp.RULE_PHI_LUT):
        o3 = bp.decode(tc, lam, pack_bits(s), 2 * tc.m + 2, early_term=False, prec=32, rule=rule)
        clear = np.abs(ref) > 1e-2
        assert (o3["bits"][clear] == (ref[clear] < 0)).all()


@pytest.mark.parametrize("seed", range(6))
def test_tree_codes_no_skip_equal_bitwise_map(seed):
    """The "without skipping" variant (Table 1 left columns, R26) is the same BP
    (a degree-1 VN's extrinsic message is lambda: Eq. (4) with an empty sum), so on a
    cycle-free graph it also reaches the brute-force bitwise MAP posterior."""
    rng = np.random.default_rng(300 + seed)
    tc = tree_code(rng, n_cn=int(rng.integers(2, 6)))
    assert (tc.vn_degree == 1).any()
    lam = rng.normal(0.4, 1.5, tc.n)
    s = rng.integers(0, 2, tc.m)
    ref = brute.bitwise_map(tc.dense(), s, lam)
    o = bp.decode(tc, lam, pack_bits(s), 2 * tc.m + 2, early_term=False, prec=64, posterior=True, no_skip=True)
    assert np.allclose(o["post"], ref, atol=1e-9, rtol=1e-9)
    E_it, n_a = bp.graph_sizes(tc, no_skip=True)
    assert (E_it, n_a) == (tc.num_edges, tc.n)


def test_no_skip_equals_skip_in_fp64(code_c1):
    """M2: skipping degree-1 VNs changes the work, not the messages: every
    active-edge message and active posterior agree to rounding, and the degree-1 edges'
    stored messages are the CN outputs the skipping decoder folds into its decisions."""
    f = gen_frame(code_c1, 0.2, 5, 0)
    lam = bp.llr_from_md_f64(f["v"], f["xnorm"], 0.2)
    a = bp.decode(code_c1, lam, f["synd"], 25, early_term=False, prec=64, trace=True)
    b = bp.decode(code_c1, lam, f["synd"], 25, early_term=False, prec=64, trace=True, no_skip=True)
    assert (a["bits"] == b["bits"]).all() and a["iters"] == b["iters"] and a["converged"] == b["converged"]
    act_e = np.nonzero(code_c1.vn_degree[code_c1.edge_vn] >= 2)[0]
    act_v = np.nonzero(code_c1.vn_degree >= 2)[0]
    assert np.allclose(b["r_trace"][:, act_e], a["r_trace"], rtol=1e-9, atol=1e-9)
    assert np.allclose(b["L_trace"][:, act_v], a["L_trace"], rtol=1e-9, atol=1e-9)


def test_loopy_tiny_codes_vs_ml():
    """S:223 / S:485: on n <= 16 codes, a converged BP output lies in the coset
    and its likelihood never exceeds the block-ML member's; with at most one
    weak erroneous prior symbol BP converges to the ML word >= 95% of the time."""
    rng = np.random.default_rng(7)
    agree = conv = trials = 0
    for t in range(60):
        n = int(rng.integers(8, 15))
        code = random_code(n, int(rng.integers(3, n // 2 + 2)), rng, frac_deg1=0.3)
        h = code.dense()
        u = rng.integers(0, 2, n).astype(np.uint8)
        s = (h.astype(int) @ u) % 2
        lam = (1.0 - 2.0 * u) * rng.uniform(2.0, 4.0, n)
        k = int(rng.integers(0, n))
        lam[k] = -0.3 * np.sign(lam[k])          # one weak erroneous symbol
        o = bp.decode(code, lam, pack_bits(s), 50, early_term=True, prec=64)
        ml, ml_ll = brute.block_ml(h, s, lam)
        trials += 1
        if o["converged"]:
            conv += 1
            assert ((h.astype(int) @ o["bits"]) % 2 == s).all()
            assert brute.log_likelihood(o["bits"], lam) <= ml_ll + 1e-9
            agree += int((o["bits"] == ml).all())
    assert conv / trials >= 0.95 and agree == conv


@pytest.mark.parametrize("prec", [32, 64])
def test_zero_noise_converges_in_one_iteration(code_c1, prec):
    """Noiseless input converges at l = 1 with c = u (BASELINE north_star)."""
    f = gen_frame(code_c1, 0.161, 9, 0)
    lam = (1.0 - 2.0 * f["u"].astype(np.float64)) * 8.0
    o = bp.decode(code_c1, lam, f["synd"], 100, early_term=True, prec=prec)
    assert o["converged"] and o["iters"] == 1 and (o["bits"] == f["u"]).all()


@pytest.mark.parametrize("rule", [bp.RULE_EXACT, bp.RULE_PHI_LUT])
def test_coset_translation_symmetry_bit_exact(code_c1, rule):
    """decode(lambda * (1-2e), S xor He) = decode(lambda, S) xor e, with the same
    iteration count and identical |messages| -- bit-exact in fp32 because every
    step is odd-symmetric and IEEE rounding commutes with negation.  Pins the
    syndrome sign of the CN rule (reading R1) against a plain invariant."""
    rng = np.random.default_rng(3)
    for fid, snr in [(0, 0.161), (1, 0.25), (2, 0.4)]:
        f = gen_frame(code_c1, snr, 1, fid)
        lam = bp.llr_from_md_f32(f["v"], f["xnorm"], snr)
        e = rng.integers(0, 2, code_c1.n).astype(np.uint8)
        se = bp.syndrome(code_c1, e)
        from synth.frames import unpack_bits
        s0 = unpack_bits(f["synd"], code_c1.m)
        a = bp.decode(code_c1, lam, f["synd"], 40, rule=rule, prec=32, trace=True)
        b = bp.decode(code_c1, (lam * (1 - 2.0 * e)).astype(np.float32), pack_bits(s0 ^ se), 40,
                      rule=rule, prec=32, trace=True)
        assert a["iters"] == b["iters"] and a["converged"] == b["converged"]
        assert ((a["bits"] ^ e) == b["bits"]).all()
        assert np.array_equal(np.abs(a["r_trace"]), np.abs(b["r_trace"]))


def test_domain_equivalence_ratio_vs_llr():
    """S:218 / S:487: the literal ratio-domain Eqs. (1)-(5) (M1, every VN
    updated) and the LLR sign/phi form with degree-1 skip (M2) give identical
    decisions; posteriors agree to 1e-9 where the ratio domain is well
    conditioned (|LLR| < 12) -- also the degree-1-skip equivalence."""
    rng = np.random.default_rng(11)
    for t in range(150):
        n = int(rng.integers(6, 13))
        code = random_code(n, int(rng.integers(3, 7)), rng, frac_deg1=0.5)
        if (code.cn_degree < 2).any():
            continue
        lam = rng.normal(0.5, 1.2, n)
        s = rng.integers(0, 2, code.m)
        it = int(rng.integers(1, 7))
        o2 = bp.decode(code, lam, pack_bits(s), it, early_term=False, prec=64, posterior=True)
        o1 = literal.decode_ratio(code.dense(), lam, s, it, early_term=False)
        assert (o1["bits"] == o2["bits"]).all()
        ok = np.abs(o2["post"]) < 12
        assert np.allclose(o1["post"][ok], o2["post"][ok], atol=1e-9, rtol=1e-9)


# ----------------------------------------------------------------- fp32 replay vs fp64 definition

@pytest.mark.parametrize("rule", [bp.RULE_EXACT, bp.RULE_PHI_LUT])
def test_m3_teacher_forced_vs_m2(code_c1, rule):
    """BASELINE north_star tolerance |dLLR| <= 1e-3 max(1, |LLR|) per iteration:
    from the fp32 state (r^{l-1}, L^{l-1}) one fp64 step must land within the
    tolerance of the fp32 state (r^l, L^l), every l, on converging and
    non-converging frames."""
    for fid, snr in [(0, 0.161), (1, 0.3)]:
        f = gen_frame(code_c1, snr, 2, fid)
        lam32 = bp.llr_from_md_f32(f["v"], f["xnorm"], snr)
        o = bp.decode(code_c1, lam32, f["synd"], 60, early_term=True, rule=rule, prec=32, trace=True)
        E_it, n_a = bp.graph_sizes(code_c1)
        r_prev = np.zeros(E_it)
        act = np.diff(code_c1.vn_ptr) >= 2
        L_prev = lam32.astype(np.float64)[act]
        for l in range(o["iters"]):
            r64, L64 = bp.step64(code_c1, lam32, f["synd"], r_prev, L_prev, rule=rule)
            r32, L32 = o["r_trace"][l].astype(np.float64), o["L_trace"][l].astype(np.float64)
            assert (np.abs(r64 - r32) <= 1e-3 * np.maximum(1, np.abs(r64))).all(), l
            assert (np.abs(L64 - L32) <= 1e-3 * np.maximum(1, np.abs(L64))).all(), l
            r_prev, L_prev = r32, L32


def test_m3_matches_m2_on_converging_frames(code_c1):
    rng_ok = 0
    for fid in range(6):
        f = gen_frame(code_c1, 0.35, 4, fid)
        lam = bp.llr_from_md_f32(f["v"], f["xnorm"], 0.35)
        a = bp.decode(code_c1, lam, f["synd"], 100, prec=32)
        b = bp.decode(code_c1, lam, f["synd"], 100, prec=64)
        assert a["converged"] == b["converged"]
        if a["converged"]:
            rng_ok += 1
            assert (a["bits"] == b["bits"]).all() and (a["bits"] == f["u"]).all()
    assert rng_ok >= 4


def test_convergence_soundness_and_early_term_modes(code_c1):
    """converged => H c = S_B; ET off runs exactly N iterations."""
    from synth.frames import unpack_bits
    for fid, snr in [(0, 0.161), (1, 0.3)]:
        f = gen_frame(code_c1, snr, 5, fid)
        lam = bp.llr_from_md_f32(f["v"], f["xnorm"], snr)
        s = unpack_bits(f["synd"], code_c1.m)
        for et in (True, False):
            o = bp.decode(code_c1, lam, f["synd"], 30, early_term=et, prec=32)
            assert o["converged"] == bool((bp.syndrome(code_c1, o["bits"]) == s).all())
            if not et:
                assert o["iters"] == 30


def test_non_finite_frame_is_invalid(code_c1):
    f = gen_frame(code_c1, 0.3, 0, 0)
    lam = bp.llr_from_md_f32(f["v"], f["xnorm"], 0.3)
    lam[17] = np.nan
    o = bp.decode(code_c1, lam, f["synd"], 10, prec=32)
    assert o["iters"] == -1 and not o["converged"] and not o["bits"].any()


def test_determinism(code_c1):
    f = gen_frame(code_c1, 0.161, 0, 3)
    lam = bp.llr_from_md_f32(f["v"], f["xnorm"], 0.161)
    a = bp.decode(code_c1, lam, f["synd"], 20, prec=32, trace=True)
    b = bp.decode(code_c1, lam, f["synd"], 20, prec=32, trace=True)
    assert np.array_equal(a["r_trace"], b["r_trace"]) and np.array_equal(a["bits"], b["bits"])


# ----------------------------------------------------------------- LLR from MD output (reading R13)

def test_llr_from_md_properties():
    """v = 0 -> 0, sign(lambda) = sign(v); fp32 and fp64 agree; the
    calibration of reading R13 is checked statistically in test_synth."""
    rng = np.random.default_rng(1)
    v = rng.normal(0, 0.4, 4096).astype(np.float32)
    v[:8] = 0
    xn = np.abs(rng.normal(2.8, 0.3, 512)).astype(np.float32)
    a = bp.llr_from_md_f32(v, xn, 0.161)
    b = bp.llr_from_md_f64(v, xn, 0.161)
    assert (a[:8] == 0).all()
    assert (np.sign(a) == np.sign(v)).all()
    assert np.allclose(a, b, rtol=2e-6, atol=1e-7)
    # closed form at one point: snr = 1 -> c = 2 sqrt(2); xnorm NULL -> sqrt(8)
    one = bp.llr_from_md_f64(np.array([0.5] * 8), None, 1.0)
    assert one[0] == pytest.approx(2 * math.sqrt(2) * math.sqrt(8) * 0.5, rel=1e-15)


# ----------------------------------------------------------------- MD front end (N6)

@pytest.mark.parametrize("d", [1, 2, 4, 8])
def test_md_product_table_and_alice_llr(d):
    """The oracle's division-algebra table reproduces synth's independent Cayley-Dickson
    product; lambda = c (alpha x) equals the normalised form c |x| (alpha x^) of R13 up to
    fp32 rounding (M(alpha) is linear), and noiseless blocks give lambda = c |y| u~."""
    from synth.frames import cd_mul, md_alice, md_bob
    rng = np.random.default_rng(d)
    a = rng.standard_normal((500, d))
    b = rng.standard_normal((500, d))
    k, s = bp.md_table(d)
    got = np.zeros_like(a)
    for i in range(d):
        for q in range(d):
            got[:, i] += s[i, q] * a[:, k[i, q]] * b[:, q]
    assert np.abs(got - cd_mul(a, b)).max() < 1e-12
    n = 64 * d
    x = rng.standard_normal(n)
    u = rng.integers(0, 2, n).astype(np.uint8)
    y = x + rng.standard_normal(n) * 2.0
    alpha = md_bob(y, u, d).reshape(-1)
    snr = 0.161
    lam = bp.md_alice_f32(x.astype(np.float32), alpha.astype(np.float32), snr, d).astype(np.float64)
    v, xn = md_alice(x, alpha.reshape(-1, d), d)
    ref = 2 * math.sqrt(snr * (1 + snr)) * np.repeat(xn, d) * v
    assert np.allclose(lam, ref, rtol=1e-5, atol=1e-5)
    # noiseless: x = y -> alpha x = |y| u~
    alpha0 = md_bob(x, u, d).reshape(-1)
    lam0 = bp.md_alice_f32(x.astype(np.float32), alpha0.astype(np.float32), snr, d).astype(np.float64)
    xn0 = np.repeat(np.linalg.norm(x.reshape(-1, d), axis=1), d)
    assert np.allclose(lam0, 2 * math.sqrt(snr * (1 + snr)) * xn0 * (1 - 2.0 * u) / math.sqrt(d), rtol=1e-5, atol=1e-5)


# ----------------------------------------------------------------- degree-1 decision (N1)

def _two_check_code():
    """VNs 0-2 of degree 2 on CN 0 and CN 1 (active), VN 3 degree-1 on CN 0, VN 4 on CN 1."""
    h = np.array([[1, 1, 1, 1, 0],
                  [1, 1, 1, 0, 1]], np.uint8)
    return from_dense(h)


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("rule", [bp.RULE_EXACT, bp.RULE_PHI_LUT])
def test_degree1_decision_is_posterior_sign(prec, rule):
    """Step 5 ("c_i = 1 if q_i > 1") for a degree-1 VN after one iteration: its
    posterior ratio is q^0 times the CN ratio (Eq. 5 with one factor), i.e. the LLR
    lambda_d + 2 atanh(sigma prod tanh(lambda_a / 2)) -- the closed form of Eqs. (2)-(3),
    evaluated here in fp64 without phi.  Away from ties every precision and rule must give
    its sign, including the fp32 replay's phi-domain comparison (S_k < p_k)."""
    code = _two_check_code()
    rng = np.random.default_rng(7)
    checked = 0
    for t in range(400):
        lam = rng.normal(0.0, 3.0, 5) * rng.choice([0.05, 1.0, 4.0], 5)
        s0 = int(rng.integers(0, 2))
        t_prod = np.prod(np.tanh(lam[:3] / 2.0)) * (1 - 2 * s0)
        rho = 2.0 * np.arctanh(np.clip(t_prod, -1 + 1e-16, 1 - 1e-16))
        post = lam[3] + rho
        if abs(rho) > 25 or abs(post) < 0.05 * max(1.0, abs(lam[3])):
            continue   # fp32 saturation / near-tie: the sign is not fixed by the closed form
        o = bp.decode(code, lam, pack_bits([s0, 0]), 1, early_term=False, rule=rule, prec=prec)
        assert int(o["bits"][3]) == int(post < 0), (t, lam, s0)
        checked += 1
    assert checked > 200


def test_degree1_decision_unclamped():
    """R6 clamps stored messages only: a degree-1 VN with lambda = -30.5 whose CN output is
    about +30.9 (three inputs of 32: rho = 2 atanh(tanh(16)^3) = 30.9) has a positive
    posterior -> bit 0, although the clamped message 30 would give -0.5 -> bit 1."""
    code = _two_check_code()
    lam = np.array([32.0, 32.0, 32.0, -30.5, 1.0])
    # tanh(16) rounds to 1 in double, so take the phi form of the same closed form
    rho = bp.phi_def(3 * bp.phi_def(32.0))
    assert 30.5 < rho < 31.0
    for prec in (32, 64):
        for rule in (bp.RULE_EXACT, bp.RULE_PHI_LUT):
            o = bp.decode(code, lam, pack_bits([0, 0]), 1, early_term=False, rule=rule, prec=prec)
            assert int(o["bits"][3]) == 0, (prec, rule)


# ----------------------------------------------------------------- 16-bit message storage (R28 / N7)

@pytest.mark.parametrize("rule", [bp.RULE_EXACT, bp.RULE_PHI_LUT])
def test_msg16_teacher_forced_vs_m2(code_c1, rule):
    """BASELINE north_star tolerance with 16-bit stored messages: from the M3-msg16
    state (stored r^{l-1}, L^{l-1}) one fp64 step of the plain definition (M2) lands
    within |dLLR| <= 1e-3 max(1, |LLR|) of the stored r^l and of L^l, every l, on
    converging and non-converging frames (the storage rounding is <= 2^-11 < 1e-3)."""
    for fid, snr in [(0, 0.161), (1, 0.3), (2, 0.22)]:
        f = gen_frame(code_c1, snr, 2, fid)
        lam32 = bp.llr_from_md_f32(f["v"], f["xnorm"], snr)
        o = bp.decode(code_c1, lam32, f["synd"], 60, rule=rule, prec=32, trace=True, msg16=True)
        E_it, n_a = bp.graph_sizes(code_c1)
        r_prev = np.zeros(E_it)
        act = np.diff(code_c1.vn_ptr) >= 2
        L_prev = lam32.astype(np.float64)[act]
        worst = 0.0
        for l in range(o["iters"]):
            r64, L64 = bp.step64(code_c1, lam32, f["synd"], r_prev, L_prev, rule=rule)
            r16, L32 = o["r_trace"][l].astype(np.float64), o["L_trace"][l].astype(np.float64)
            dr = np.abs(r64 - r16) / np.maximum(1, np.abs(r64))
            assert (dr <= 1e-3).all(), (l, dr.max())
            assert (np.abs(L64 - L32) <= 1e-3 * np.maximum(1, np.abs(L64))).all(), l
            worst = max(worst, dr.max())
            r_prev, L_prev = r16, L32
        assert worst > 1e-4   # the rounding is visible (a stored fp32 copy would sit near 1e-6)


def test_msg16_storage_grid_and_first_iteration(code_c1):
    """N7: every stored message is an integer multiple of 2^-10 of magnitude <= 30 and
    lies within 2^-11 of the fp32 decoder's message at l = 1 (identical inputs x = lambda
    there); the posterior of l = 1 is the fp32 decoder's exactly, because the VN sum is
    taken over the unrounded outputs (Eq. (4) of the current iteration)."""
    f = gen_frame(code_c1, 0.161, 5, 0)
    lam = bp.llr_from_md_f32(f["v"], f["xnorm"], 0.161)
    a = bp.decode(code_c1, lam, f["synd"], 5, early_term=False, prec=32, trace=True)
    b = bp.decode(code_c1, lam, f["synd"], 5, early_term=False, prec=32, trace=True, msg16=True)
    q = b["r_trace"].astype(np.float64) * 1024.0
    assert (q == np.round(q)).all() and (np.abs(q) <= 30720).all()
    assert (np.abs(b["r_trace"][0].astype(np.float64) - a["r_trace"][0]) <= 2.0 ** -11).all()
    assert np.array_equal(a["L_trace"][0], b["L_trace"][0])
    assert not np.array_equal(a["r_trace"][0], b["r_trace"][0])


@pytest.mark.parametrize("rule", [bp.RULE_EXACT, bp.RULE_PHI_LUT])
def test_msg16_coset_translation_symmetry_bit_exact(code_c1, rule):
    """The coset-translation symmetry (pins R1) survives the storage rounding: rint is
    odd-symmetric (ties to even), so flipping lambda's signs on a coset translate flips
    the stored messages exactly."""
    from synth.frames import unpack_bits
    rng = np.random.default_rng(4)
    for fid, snr in [(0, 0.161), (1, 0.3)]:
        f = gen_frame(code_c1, snr, 6, fid)
        lam = bp.llr_from_md_f32(f["v"], f["xnorm"], snr)
        e = rng.integers(0, 2, code_c1.n).astype(np.uint8)
        s0 = unpack_bits(f["synd"], code_c1.m)
        a = bp.decode(code_c1, lam, f["synd"], 40, rule=rule, prec=32, trace=True, msg16=True)
        b = bp.decode(code_c1, (lam * (1 - 2.0 * e)).astype(np.float32), pack_bits(s0 ^ bp.syndrome(code_c1, e)),
                      40, rule=rule, prec=32, trace=True, msg16=True)
        assert a["iters"] == b["iters"] and a["converged"] == b["converged"]
        assert ((a["bits"] ^ e) == b["bits"]).all()
        assert np.array_equal(np.abs(a["r_trace"]), np.abs(b["r_trace"]))


def test_msg16_zero_noise_and_tree_map():
    """Noiseless input converges at l = 1 with c = u; on cycle-free codes the
    decisions equal the brute-force bitwise MAP decisions (BP exact on trees) wherever
    |MAP LLR| is clear of the storage rounding."""
    from synth.codes import make_met_code
    code = make_met_code("r0.1", 2048)
    f = gen_frame(code, 0.161, 9, 1)
    lam = ((1.0 - 2.0 * f["u"].astype(np.float64)) * 8.0).astype(np.float32)
    o = bp.decode(code, lam, f["synd"], 100, prec=32, msg16=True)
    assert o["converged"] and o["iters"] == 1 and (o["bits"] == f["u"]).all()
    for seed in range(8):
        rng = np.random.default_rng(500 + seed)
        tc = tree_code(rng, n_cn=int(rng.integers(2, 6)))
        lam = rng.normal(0.4, 1.5, tc.n).astype(np.float32)
        s = rng.integers(0, 2, tc.m)
        ref = brute.bitwise_map(tc.dense(), s, lam.astype(np.float64))
        for rule in (bp.RULE_EXACT, bp.RULE_PHI_LUT):
            o3 = bp.decode(tc, lam, pack_bits(s), 2 * tc.m + 2, early_term=False, prec=32, rule=rule, msg16=True)
            clear = np.abs(ref) > 2e-2
            assert (o3["bits"][clear] == (ref[clear] < 0)).all()


def test_msg16_decodes_like_fp32_storage(code_c1):
    """Converging frames decode to u with 16-bit storage as with fp32 storage, in about
    the same number of iterations (the rounding is far below the channel noise)."""
    n_ok, d_it = 0, []
    for fid in range(8):
        f = gen_frame(code_c1, 0.35, 7, fid)
        lam = bp.llr_from_md_f32(f["v"], f["xnorm"], 0.35)
        a = bp.decode(code_c1, lam, f["synd"], 100, prec=32)
        b = bp.decode(code_c1, lam, f["synd"], 100, prec=32, msg16=True)
        assert a["converged"] == b["converged"]
        if b["converged"]:
            n_ok += 1
            assert (b["bits"] == f["u"]).all()
            d_it.append(abs(a["iters"] - b["iters"]))
    assert n_ok >= 6 and max(d_it) <= 2
