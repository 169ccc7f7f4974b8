"""Report arithmetic of the paper's tables and the roofline byte model.

* capacity / beta: reconciliation efficiency beta = R / C(SNR),
  C = 1/2 log2(1 + SNR) -- reproduces Table 1's 93.40 / 95.84 / 96.99 %
  (PAPER.md lines 57-58).
* throughput_from_latency: "Error Correction Speed" = n / (N * latency per
  iteration per codeword) -- reproduces Table 1's six speeds (PAPER.md 69-72).
* algorithmic bytes per codeword-iteration (DESIGN.md
  "Roofline"): what one flooding iteration must move at minimum, and what
  each of this build's kernels moves by design.
"""
from __future__ import annotations

import math


def capacity(snr: float) -> float:
    return 0.5 * math.log2(1.0 + snr)


def beta(rate: float, snr: float) -> float:
    return rate / capacity(snr)


def throughput_from_latency(n: int, iters: int, latency_s: float) -> float:
    """bits/s = n / (N * latency_per_iteration_per_codeword)."""
    return n / (iters * latency_s)


def bytes_per_cw_iter(E_it: int, n_1: int, n_a: int, m: int, s: int = 4, s_r: int | None = None) -> dict:
    """Byte model per codeword-iteration (fp32 node arrays, s = 4 bytes; edge messages of
    s_r bytes, 4 = fp32 or 2 = the 16-bit storage of DESIGN.md N7).

    alg      : the method's floor -- each iterating edge message read once and
               written once, each degree-1 prior read once, each active VN
               prior read once and posterior written once and read once, plus
               the syndrome bits: 2 E_it s_r + s(n_1 + 3 n_a) + m/8.
    cn       : this build's check-node pass -- r read + r written (2 E_it s_r),
               degree-1 priors (n_1 s), posterior L read once (n_a s; the
               E_it gathers are L2 hits by design), syndrome bits (m/8).
    vn       : this build's variable-node pass -- r read again (E_it s_r),
               prior and posterior of every active VN (2 n_a s).
    two_pass : cn + vn.
    """
    s_r = s if s_r is None else s_r
    alg = 2 * E_it * s_r + s * (n_1 + 3 * n_a) + m / 8.0
    cn = 2 * E_it * s_r + s * (n_1 + n_a) + m / 8.0
    vn = E_it * s_r + s * 2 * n_a
    return {"alg": alg, "cn": cn, "vn": vn, "two_pass": cn + vn}
