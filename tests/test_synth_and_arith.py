"""Pins of the input generators and the report arithmetic against PAPER.md numbers."""
import json
import math
from pathlib import Path

import numpy as np
import pytest

from paper_1711_01783_b200 import metrics
from synth.codes import make_met_code, met_counts
from synth.frames import (cd_mul, gen_frame, left_mul_matrix, md_alice, md_bob, pack_bits,
                          unpack_bits)

T1 = json.loads((Path(__file__).parent / "golden" / "table1.json").read_text())


@pytest.mark.parametrize("col", T1["columns"], ids=lambda c: f"rate{c['rate']}")
def test_beta_table1(col):
    """beta = R / C(SNR), C = 1/2 log2(1+SNR): Table 1 row 'beta'."""
    assert 100 * metrics.beta(col["rate"], col["snr"]) == pytest.approx(col["beta_pct"], abs=0.01)


@pytest.mark.parametrize("col", T1["columns"], ids=lambda c: f"rate{c['rate']}")
@pytest.mark.parametrize("mode", ["noskip", "skip"])
def test_speed_table1(col, mode):
    """speed = n / (N * latency per iteration): Table 1 rows 'Latency' and 'Speed'."""
    bps = metrics.throughput_from_latency(T1["n"], col["iters"], col["latency_ms"][mode] * 1e-3)
    assert bps / 1e6 == pytest.approx(col["speed_mbps"][mode], abs=0.05)


@pytest.mark.parametrize("col", T1["columns"], ids=lambda c: f"rate{c['rate']}")
def test_structural_arithmetic_table1(col):
    """CNs = n(1-R); iterating edges = total edges - ignored (degree-1) VNs."""
    assert round(T1["n"] * (1 - col["rate"])) == col["updated_cns"]
    assert col["total_edges"] - col["ignored_vns"] == col["iter_edges"]


@pytest.mark.parametrize("family,idx", [("r0.1", 0), ("r0.1de", 0), ("r0.05", 1), ("r0.02", 2)])
def test_standin_codes_match_table1(family, idx):
    """The stand-in ensembles reproduce every structural count of Table 1 at n = 10^6."""
    col = T1["columns"][idx]
    c = make_met_code(family, T1["n"])
    st = c.stats()
    assert st["edges"] == col["total_edges"]
    assert st["m"] == col["updated_cns"]
    assert st["n_deg1"] == col["ignored_vns"]
    assert st["n_active"] == T1["n"] - col["ignored_vns"]
    assert st["iter_edges"] == col["iter_edges"]
    # no parallel edges, canonical CSR/CSC consistency
    key = c.edge_cn().astype(np.int64) * c.n + c.edge_vn
    assert np.unique(key).size == key.size
    assert np.array_equal(np.sort(c.vn_edge), np.arange(c.num_edges))
    assert np.array_equal(c.edge_vn[c.vn_edge], np.repeat(np.arange(c.n), c.vn_degree))


def test_standin_small_sizes():
    """SURVEY App. B general-n formulas: C1 / C2 shapes."""
    for n, m, E, E_it in [(2048, 1843, 7716, 5924), (65536, 58982, 246907, 189563)]:
        st = make_met_code("r0.1", n).stats()
        assert (st["m"], st["edges"], st["iter_edges"]) == (m, E, E_it)
    assert met_counts("r0.1", 10 ** 6)["core_deg"] == {10: 7500, 11: 17500}


def test_r01de_degree_structure():
    """DESIGN.md R29: the density-evolution stand-in at n = 10^6 has exactly the degree
    distribution its DE threshold was computed for (tools/met_de.py R01DE)."""
    c = make_met_code("r0.1de", 10 ** 6)
    vd, cd = c.vn_degree, c.cn_degree
    got = dict(zip(*[x.tolist() for x in np.unique(vd, return_counts=True)]))
    # active VNs: (core 2, inner 21) 50,000 -> 23; (3, 21) 17,500 -> 24; (3, 20) 57,500 -> 23
    assert got == {1: 875000, 23: 50000 + 57500, 24: 17500}
    got = dict(zip(*[x.tolist() for x in np.unique(cd, return_counts=True)]))
    assert got == {3: 57500, 4: 817500, 13: 25000}
    # no 4-cycles: no two VNs share two checks
    ec = c.edge_cn()
    keys = []
    for j in np.flatnonzero(cd >= 2)[:200000:7]:
        vs = np.sort(c.edge_vn[c.cn_ptr[j]:c.cn_ptr[j + 1]])
        iu, ju = np.triu_indices(vs.size, 1)
        keys.append(vs[iu].astype(np.int64) << 32 | vs[ju])
    keys = np.concatenate(keys)
    assert np.unique(keys).size == keys.size


def test_biawgn_frames():
    """DESIGN.md R31: lambda = 2 snr y, y = (1 - 2u) + N(0, 1/snr), so lambda is a consistent
    Gaussian LLR, N(+-2 snr, 4 snr); S_B = H u; reproducible per (key, frame)."""
    from synth.frames import gen_frame_biawgn
    code = make_met_code("r0.1", 65536)
    a = gen_frame_biawgn(code, 0.161, 3, 7)
    b = gen_frame_biawgn(code, 0.161, 3, 7)
    assert np.array_equal(a["llr"], b["llr"]) and np.array_equal(a["synd"], b["synd"])
    sgn = 1.0 - 2.0 * a["u"]
    t = a["llr"].astype(np.float64) * sgn
    assert abs(t.mean() - 2 * 0.161) < 0.01 and abs(t.var() - 4 * 0.161) < 0.02
    from oracle import bp
    assert np.array_equal(bp.syndrome(code, a["u"]), unpack_bits(a["synd"], code.m))


def test_density_evolution_thresholds():
    """SURVEY 8(f) #4 / DESIGN.md R29: discretised DE (tools/met_de.py) converges at the
    headline SNR 0.161 for the r0.1de ensemble and not for the Table-1-count stand-in r0.1
    (DE threshold 0.182, matching its measured waterfall, profiles/r1_c5_fer_sweep.jsonl)."""
    import sys
    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1] / "tools"))
    import met_de
    ok_de, _, _ = met_de.de(met_de.R01DE, 0.161, iters=400)
    ok_r01, _, _ = met_de.de(met_de.R01_STANDIN, 0.161, iters=400)
    assert ok_de and not ok_r01


def test_code_generation_deterministic(tmp_path, monkeypatch):
    a = make_met_code("r0.1", 2048, cache=False)
    b = make_met_code("r0.1", 2048, cache=False)
    assert np.array_equal(a.edge_vn, b.edge_vn) and np.array_equal(a.cn_ptr, b.cn_ptr)


# ----------------------------------------------------------------- multidimensional reconciliation

@pytest.mark.parametrize("d", [1, 2, 4, 8])
def test_md_rotation_identities(d):
    """M(alpha) y^ = u~ to 1e-10, |alpha| = 1, M orthogonal,
    {A_k w} orthonormal; noiseless x = y gives v = u~ exactly."""
    rng = np.random.default_rng(d)
    y = rng.standard_normal(d * 2000)
    u = rng.integers(0, 2, d * 2000).astype(np.uint8)
    al = md_bob(y, u, d)
    assert np.allclose(np.linalg.norm(al, axis=1), 1.0, atol=1e-12)
    v, xn = md_alice(y, al, d)
    assert np.abs(v - (1 - 2.0 * u) / math.sqrt(d)).max() < 1e-10
    for k in range(20):
        M = left_mul_matrix(al[k])
        assert np.allclose(M @ M.T, np.eye(d), atol=1e-12)
        w = rng.standard_normal(d)
        w /= np.linalg.norm(w)
        basis = np.stack([cd_mul(np.eye(d)[i], w) for i in range(d)])
        assert np.allclose(basis @ basis.T, np.eye(d), atol=1e-12)


def test_frames_reproducible_and_syndrome():
    code = make_met_code("r0.1", 2048)
    a = gen_frame(code, 0.161, 3, 17)
    b = gen_frame(code, 0.161, 3, 17)
    assert np.array_equal(a["v"], b["v"]) and np.array_equal(a["synd"], b["synd"])
    s = unpack_bits(a["synd"], code.m)
    h = code.dense().astype(int)
    assert np.array_equal((h @ a["u"]) % 2, s)
    assert np.array_equal(unpack_bits(pack_bits(s), code.m), s)


def test_llr_calibration_reading_r13():
    """Reading R13: lambda = 2 sqrt(snr(1+snr)) |x| v is a calibrated BIAWGN LLR
    for MD output: E[sign * lambda] ~ var/2 ~ 2 snr and slope of the empirical
    LLR on lambda ~ 1 (X2 in SURVEY App. A)."""
    code = make_met_code("r0.1", 65536)
    snr = 0.161
    f = gen_frame(code, snr, 0, 0)
    lam = 2 * math.sqrt(snr * (1 + snr)) * np.repeat(f["xnorm"], 8).astype(np.float64) * f["v"]
    sgn = 1 - 2.0 * f["u"]
    t = lam * sgn
    assert abs(t.mean() - 2 * snr) < 0.03 and abs(t.var() / 2 - 2 * snr) < 0.03
    bins = np.linspace(-2.5, 2.5, 21)
    idx = np.digitize(lam, bins)
    xs, ys = [], []
    for b in range(1, len(bins)):
        sel = idx == b
        if sel.sum() > 500:
            xs.append(lam[sel].mean())
            ys.append(2 * np.arctanh(np.clip(sgn[sel].mean(), -0.999, 0.999)))
    slope = np.polyfit(xs, ys, 1)[0]
    assert 0.85 < slope < 1.15


def test_byte_model_survey_numbers():
    """rate-0.1 algorithmic floor 28.25 MB, two-pass 39.82 MB per codeword-iteration."""
    bm = metrics.bytes_per_cw_iter(2892500, 875000, 125000, 900000)
    assert bm["alg"] / 1e6 == pytest.approx(28.25, abs=0.01)
    assert bm["two_pass"] / 1e6 == pytest.approx(39.82, abs=0.01)
