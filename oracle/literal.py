"""M1: PAPER.md Eqs. (1)-(5) written out literally (TEST INFRASTRUCTURE).

Ratio domain, float64, pure-Python loops, every VN updated (no degree-1 skip),
direct extrinsic products exactly as printed -- for tiny codes only.  It is the
cross-check that the LLR sign/phi form of oracle/bp_oracle.c (M2) computes the
paper's rule.

  Eq. (1)  q^0_i = q^0(1)/q^0(0) = exp(-lambda_i)
  Eq. (3)  t = prod_{i' in R_j \\ i} (1 - q_{i'j}) / (1 + q_{i'j})
           multiplied by sigma_j = 1 - 2 S_B[j]  (reading R1)
  Eq. (2)  r_ji = (1 - t)/(1 + t)
  Eq. (4)  q_ij = q^0_i prod_{j' in C_i \\ j} r_{j'i}
  Eq. (5)  q_i  = q^0_i prod_{j in C_i} r_ji; c_i = 1 iff q_i > 1
  Step 5   stop when S_A = H c^T equals S_B or l = N

r is kept in [e^-30, e^30], the ratio image of the LLR clamp |r| <= 30
(reading R6), so M1 and M2 see the same saturation.
"""
from __future__ import annotations

import math

import numpy as np

R_LO, R_HI = math.exp(-30.0), math.exp(30.0)


def decode_ratio(h: np.ndarray, llr, synd_bits, max_iter: int, early_term: bool = True):
    h = np.asarray(h)
    m, n = h.shape
    R = [[i for i in range(n) if h[j, i]] for j in range(m)]      # R_j
    Cn = [[j for j in range(m) if h[j, i]] for i in range(n)]     # C_i
    q0 = [math.exp(-float(x)) for x in llr]                       # Eq. (1)
    q = {(i, j): q0[i] for j in range(m) for i in R[j]}           # Step 2 init
    r = {}
    c = [0] * n
    post = [0.0] * n
    it = 0
    conv = False
    for l in range(1, max_iter + 1):
        # Step 3: check nodes, Eqs. (2)-(3)
        for j in range(m):
            sigma = 1.0 - 2.0 * int(synd_bits[j])
            for i in R[j]:
                t = 1.0
                for i2 in R[j]:
                    if i2 != i:
                        qq = q[(i2, j)]
                        t *= (1.0 - qq) / (1.0 + qq) if math.isfinite(qq) else -1.0
                t *= sigma
                rr = (1.0 - t) / (1.0 + t) if t != -1.0 else math.inf
                r[(j, i)] = min(max(rr, R_LO), R_HI)
        # Step 4: variable nodes, Eq. (4)
        for i in range(n):
            for j in Cn[i]:
                prod = q0[i]
                for j2 in Cn[i]:
                    if j2 != j:
                        prod *= r[(j2, i)]
                q[(i, j)] = prod
        # Step 5: posterior Eq. (5), hard decision, syndrome
        for i in range(n):
            qi = q0[i]
            for j in Cn[i]:
                qi *= r[(j, i)]
            post[i] = -math.log(qi)
            c[i] = 1 if qi > 1.0 else 0
        it = l
        sa = [sum(c[i] for i in R[j]) % 2 for j in range(m)]
        if early_term and all(sa[j] == int(synd_bits[j]) for j in range(m)):
            conv = True
            break
    if not conv:
        sa = [sum(c[i] for i in R[j]) % 2 for j in range(m)]
        conv = all(sa[j] == int(synd_bits[j]) for j in range(m))
    return {"bits": np.array(c, np.uint8), "iters": it, "converged": conv,
            "post": np.array(post)}
