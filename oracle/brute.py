"""Exhaustive coset enumeration for tiny codes (TEST INFRASTRUCTURE).

For n <= 20, enumerate every c in {0,1}^n with H c^T = S_B (the coset Alice
decodes into, PAPER.md Step 5 line 141) under the virtual BIAWGN prior
P(c_i) proportional to exp((1 - 2 c_i) lambda_i / 2), lambda = ln P(0)/P(1):

* ``bitwise_map`` -- exact a-posteriori LLR of every bit (what BP computes
  exactly on a cycle-free Tanner graph);
* ``block_ml``    -- the most likely coset member (ties -> lowest integer
  index sum_i c_i 2^i, reading R22).
"""
from __future__ import annotations

import numpy as np


def coset(h: np.ndarray, synd_bits) -> np.ndarray:
    h = np.asarray(h, np.int64)
    m, n = h.shape
    if n > 22:
        raise ValueError("brute force limited to n <= 22")
    idx = np.arange(1 << n, dtype=np.int64)
    bits = ((idx[:, None] >> np.arange(n)) & 1).astype(np.int64)
    s = (bits @ h.T) & 1
    ok = (s == np.asarray(synd_bits, np.int64)[None, :]).all(1)
    return bits[ok].astype(np.uint8)


def _logw(cs: np.ndarray, llr) -> np.ndarray:
    lam = np.asarray(llr, np.float64)
    return ((1.0 - 2.0 * cs) * lam[None, :]).sum(1) / 2.0


def bitwise_map(h, synd_bits, llr) -> np.ndarray:
    cs = coset(h, synd_bits)
    lw = _logw(cs, llr)
    mx = lw.max()
    w = np.exp(lw - mx)
    out = np.empty(cs.shape[1])
    for i in range(cs.shape[1]):
        p0 = w[cs[:, i] == 0].sum()
        p1 = w[cs[:, i] == 1].sum()
        out[i] = np.log(p0) - np.log(p1) if p0 > 0 and p1 > 0 else (np.inf if p1 == 0 else -np.inf)
    return out


def block_ml(h, synd_bits, llr):
    cs = coset(h, synd_bits)
    lw = _logw(cs, llr)
    best = np.flatnonzero(lw == lw.max())
    key = (cs[best].astype(np.int64) << np.arange(cs.shape[1])).sum(1)
    k = best[np.argmin(key)]
    return cs[k], lw[k]


def log_likelihood(c, llr) -> float:
    return float(_logw(np.asarray(c, np.uint8)[None, :], llr)[0])
