#!/usr/bin/env python
"""Discretised density evolution (DE) for the multi-edge-type (MET) stand-in ensembles --
a DESIGN TOOL for SURVEY 8(f) #4 (better stand-in ensembles), not product code.

Ensemble family (the Table-1 structure, R18 / SURVEY App. B): edge types
1 = core, 2 = inner, 3 = degree-1;
  nu = sum_d a_d x1^d x2^{b_d}  (active VNs)  +  n1 x3      (degree-1 VNs)
  mu = sum_c k_c x1^c           (core checks) +  sum_e t_e x2^e x3   (inner checks)
on a BIAWGN channel with LLR ~ N(2 s, 4 s) (s = SNR, the MD virtual channel, R13),
all-zero codeword (the decoder is symmetric: coset translation, tests/test_oracle.py).

VN updates are sums of independent LLRs (FFT convolutions on a uniform LLR grid, tails
clipped); CN updates run in the (sign, phi(|x|)) domain, where they are sums as well
(sign XOR, phi additive), on a uniform phi grid.  Threshold = smallest s at which the
bit error probability of every VN class goes to ~0 within `iters` iterations (bisection).

    python tools/met_de.py                      # threshold of the r0.1 stand-in
"""
from __future__ import annotations

import math
import sys

import numpy as np
from scipy.signal import fftconvolve

# LLR grid (messages saturate at +-XM, like the decoder's |r| <= 30 clamp, R6)
DX = 0.05
XM = 30.0
X = np.arange(-XM, XM + DX / 2, DX)
NX = X.size
I0 = NX // 2            # index of x = 0


def _boxplus_table() -> np.ndarray:
    """T[i, j] = grid index of 2 atanh(tanh(x_i / 2) tanh(x_j / 2)) (the CN rule of two inputs,
    Eqs. (2)-(3) in the LLR domain), computed in the sign / phi form for accuracy."""
    a = np.abs(X)
    with np.errstate(divide="ignore", over="ignore"):
        ph = np.where(a > 0, np.log1p(2.0 / np.expm1(np.maximum(a, 1e-300))), np.inf)
    S = ph[:, None] + ph[None, :]
    with np.errstate(divide="ignore", over="ignore", invalid="ignore"):
        mag = np.where(np.isfinite(S), np.log1p(2.0 / np.expm1(np.maximum(S, 1e-300))), 0.0)
    sign = np.sign(X)[:, None] * np.sign(X)[None, :]
    return np.clip(np.rint(sign * mag / DX) + I0, 0, NX - 1).astype(np.int32).ravel()


_T = _boxplus_table()


def channel(s: float) -> np.ndarray:
    """BIAWGN LLR density N(2 s, 4 s) on the grid (tails saturate at +-XM)."""
    from scipy.stats import norm
    m, sd = 2.0 * s, 2.0 * math.sqrt(s)
    edges = np.concatenate([[-np.inf], X[:-1] + DX / 2, [np.inf]])
    return np.diff(norm.cdf((edges - m) / sd))


def vconv(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Density of the sum of two independent LLRs on the grid (saturating at +-XM)."""
    c = np.maximum(fftconvolve(a, b), 0.0)
    out = c[I0:I0 + NX].copy()
    out[0] += c[:I0].sum()
    out[-1] += c[I0 + NX:].sum()
    return out / out.sum()   # renormalised: a mass error is amplified by the degree products otherwise


def vpow(a: np.ndarray, k: int) -> np.ndarray:
    r = None
    base = a
    while k:
        if k & 1:
            r = base if r is None else vconv(r, base)
        k >>= 1
        if k:
            base = vconv(base, base)
    if r is None:
        r = np.zeros(NX)
        r[I0] = 1.0
    return r


def cconv(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Density of the CN combination of two independent LLRs (pairwise table)."""
    out = np.bincount(_T, weights=np.outer(a, b).ravel(), minlength=NX)
    return out / out.sum()


def cpow(a: np.ndarray, k: int) -> np.ndarray:
    r = None
    base = a
    while k:
        if k & 1:
            r = base if r is None else cconv(r, base)
        k >>= 1
        if k:
            base = cconv(base, base)
    return r


def mix(parts):
    tot = sum(w for w, _ in parts)
    return sum(w * d for w, d in parts) / tot


def perr(a: np.ndarray) -> float:
    return float(a[:I0].sum() + a[I0] / 2)


def de(ens: dict, s: float, iters: int = 400, tol: float = 1e-7, verbose: bool = False):
    """Runs DE at SNR s.  Returns (converged, iterations, final error probabilities)."""
    ch = channel(s)
    act = ens["act"]          # list of (fraction of n, d core degree, b inner degree)
    core = ens["core"]        # list of (fraction of n, c)
    inner = ens["inner"]      # list of (fraction of n, e inner degree)  (each with one x3 socket)
    m1, m2 = ch.copy(), ch.copy()
    hist = []
    for it in range(1, iters + 1):
        # CN -> VN, type 1: core check of degree c, edge-perspective weight c k_c
        u1 = mix([(f * c, cpow(m1, c - 1)) for f, c in core])
        # CN -> VN, type 2: inner check x2^e x3: (e - 1) type-2 inputs + the degree-1 VN's channel LLR
        u2 = mix([(f * e, cconv(cpow(m2, e - 1), ch) if e > 1 else ch) for f, e in inner])
        # degree-1 VN posterior: channel + the inner check's output to it (e type-2 inputs)
        u3 = mix([(f, cpow(m2, e)) for f, e in inner])
        # VN -> CN
        new1, new2, pe_a = [], [], []
        for f, d, b in act:
            s2 = vpow(u2, b - 1)                        # b - 1 other type-2 inputs
            s2b = vconv(s2, u2)                          # all b type-2 inputs
            # type-1 output: channel + (d - 1) type-1 + b type-2 inputs
            base = vconv(ch, s2b) if d == 1 else vconv(vconv(ch, vpow(u1, d - 1)), s2b)
            new1.append((f * d, base))
            # type-2 output: channel + d type-1 + (b - 1) type-2 inputs
            full2 = vconv(vconv(ch, vpow(u1, d)), s2)
            new2.append((f * b, full2))
            pe_a.append((f, perr(vconv(full2, u2))))
        m1, m2 = mix(new1), mix(new2)
        pe_active = sum(f * p for f, p in pe_a) / sum(f for f, _ in pe_a)
        pe1 = perr(vconv(ch, u3))
        pe = max(pe_active, pe1)
        if verbose and (it % 20 == 0 or it < 5):
            print(f"  it {it:4d}  Pe(active) {pe_active:.3e}  Pe(deg1) {pe1:.3e}", flush=True)
        if pe < tol:
            return True, it, (pe_active, pe1)
        hist.append(pe)
        if it > 40 and pe > 0.9999 * hist[-30]:   # no progress over 30 iterations: a fixed point
            return False, it, (pe_active, pe1)
    return False, iters, (pe_active, pe1)


def threshold(ens: dict, lo: float = 0.14, hi: float = 0.22, steps: int = 8, iters: int = 600) -> float:
    for _ in range(steps):
        mid = 0.5 * (lo + hi)
        ok, it, pe = de(ens, mid, iters)
        if ok:
            hi = mid
        else:
            lo = mid
    return hi


R01_STANDIN = {
    "act": [(0.1075, 2, 21), (0.0175, 3, 21)],
    "core": [(0.0075, 10), (0.0175, 11)],
    "inner": [(0.875, 3)],
}

def make_ensemble(act, core, inner):
    """Checks the edge balance of a candidate: type 1 (sum a d = sum k c), type 2
    (sum a b = sum t e), one degree-1 VN per inner check."""
    e1v = sum(f * d for f, d, _ in act)
    e1c = sum(f * c for f, c in core)
    e2v = sum(f * b for f, _, b in act)
    e2c = sum(f * e for f, e in inner)
    assert abs(e1v - e1c) < 1e-9 and abs(e2v - e2c) < 1e-9, (e1v, e1c, e2v, e2c)
    return {"act": act, "core": core, "inner": inner}


def _thr(args):
    name, ens = args
    return name, threshold(ens)


def run_many(cands: dict, procs: int = 8) -> dict:
    from multiprocessing import Pool
    with Pool(procs) as p:
        return dict(p.map(_thr, list(cands.items())))


# DESIGN.md R29 (synth/codes.py "r0.1de"): 0.0575 n inner checks x2^2 x3, every core check
# degree 13; threshold 0.153
R01DE = {
    "act": [(0.05, 2, 21), (0.0175, 3, 21), (0.0575, 3, 20)],
    "core": [(0.025, 13)],
    "inner": [(0.0575, 2), (0.8175, 3)],
}

if __name__ == "__main__":
    s = float(sys.argv[1]) if len(sys.argv) > 1 else None
    if s:
        print(de(R01_STANDIN, s, verbose=True))
    else:
        print("threshold", threshold(R01_STANDIN))
