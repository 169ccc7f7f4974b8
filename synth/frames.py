"""Seeded CV-QKD frames after multidimensional (MD) reverse reconciliation.

Channel: X ~ N(0, sigma_X^2), Z ~ N(0, sigma_Z^2), Y = X + Z,
with sigma_X^2 = 1 and SNR = sigma_X^2 / sigma_Z^2.

MD reconciliation (details in the paper's ref. [MD]):
Bob draws his binary string U, maps each d-block to u~ = (1 - 2u)/sqrt(d) and
sends the rotation alpha = u~ * conj(y^) (division-algebra product, y^ = y/|y|)
so that M(alpha) y^ = alpha * y^ = u~; Alice applies the same rotation to her
normalised block, V = alpha * (x/|x|), the "noise form of this binary string".
Bob's syndrome S_B = H U^T (Step 1) is sent with alpha.

d in {1, 2, 4, 8}: reals, complex, quaternions, octonions via Cayley-Dickson
doubling (a1, a2)(b1, b2) = (a1 b1 - conj(b2) a2, b2 a1 + a2 conj(b1)).
Octonions are alternative, so (u~ conj(y^)) y^ = u~ |y^|^2 = u~ exactly.

Every frame is reproducible from (data_key, frame_id) alone through a
counter-based Philox generator, independent of batch, lane or GPU.
"""
from __future__ import annotations

import numpy as np

from .codes import Code


def conj(a: np.ndarray) -> np.ndarray:
    out = -a
    out[..., 0] = a[..., 0]
    return out


def cd_mul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Cayley-Dickson product over the last axis (length 1, 2, 4 or 8)."""
    d = a.shape[-1]
    if d == 1:
        return a * b
    h = d // 2
    a1, a2 = a[..., :h], a[..., h:]
    b1, b2 = b[..., :h], b[..., h:]
    return np.concatenate([cd_mul(a1, b1) - cd_mul(conj(b2), a2),
                           cd_mul(b2, a1) + cd_mul(a2, conj(b1))], axis=-1)


def left_mul_matrix(alpha: np.ndarray) -> np.ndarray:
    """M(alpha) with M(alpha) w = alpha * w, as a d x d matrix (tests)."""
    d = alpha.shape[-1]
    eye = np.eye(d)
    return np.stack([cd_mul(alpha, eye[k]) for k in range(d)], axis=-1)


def frame_rng(data_key: int, frame_id: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=(int(data_key) << 64) | int(frame_id)))


def md_bob(y: np.ndarray, u: np.ndarray, d: int) -> np.ndarray:
    """alpha per d-block: alpha = u~ * conj(y/|y|)."""
    yb = y.reshape(-1, d)
    yh = yb / np.linalg.norm(yb, axis=1, keepdims=True)
    ut = (1.0 - 2.0 * u.reshape(-1, d).astype(np.float64)) / np.sqrt(d)
    return cd_mul(ut, conj(yh))


def md_alice(x: np.ndarray, alpha: np.ndarray, d: int):
    """v = alpha * (x/|x|) per block, and |x| per block."""
    xb = x.reshape(-1, d)
    xn = np.linalg.norm(xb, axis=1)
    v = cd_mul(alpha, xb / xn[:, None])
    return v.reshape(-1), xn


def syndrome_words(code: Code, u: np.ndarray) -> np.ndarray:
    """S_B = H U^T packed LSB-first into uint32 words [ceil(m/32)] (Bob, Step 1)."""
    s = np.bitwise_xor.reduceat(u[code.edge_vn].astype(np.uint8), code.cn_ptr[:-1])
    s[np.diff(code.cn_ptr) == 0] = 0
    return pack_bits(s)


def pack_bits(bits: np.ndarray) -> np.ndarray:
    bits = np.asarray(bits, dtype=np.uint8)
    nw = (bits.size + 31) // 32
    padded = np.zeros(nw * 32, np.uint8)
    padded[:bits.size] = bits
    return np.packbits(padded, bitorder="little").view("<u4").astype(np.uint32)


def unpack_bits(words: np.ndarray, n: int) -> np.ndarray:
    w = np.ascontiguousarray(words, dtype="<u4")
    return np.unpackbits(w.view(np.uint8), bitorder="little")[:n]


def gen_frame(code: Code, snr: float, data_key: int, frame_id: int, d: int = 8) -> dict:
    """One frame: Bob's bits u, S_B, Alice's MD output v (fp32) and |x| per block."""
    n = code.n
    if n % d:
        raise ValueError("n must be divisible by d")
    g = frame_rng(data_key, frame_id)
    x = g.standard_normal(n)
    z = g.standard_normal(n) / np.sqrt(snr)
    u = g.integers(0, 2, size=n, dtype=np.uint8)
    y = x + z
    alpha = md_bob(y, u, d)
    v, xn = md_alice(x, alpha, d)
    return {"u": u, "v": v.astype(np.float32), "xnorm": xn.astype(np.float32),
            "synd": syndrome_words(code, u), "frame_id": frame_id,
            "x": x.astype(np.float32), "alpha": alpha.reshape(-1).astype(np.float32)}


def gen_batch(code: Code, snr: float, data_key: int, frame_ids, d: int = 8) -> dict:
    fr = [gen_frame(code, snr, data_key, f, d) for f in frame_ids]
    return {k: np.stack([f[k] for f in fr]) for k in ("u", "v", "xnorm", "synd", "x", "alpha")} | {
        "frame_ids": np.asarray(list(frame_ids))}


def gen_frame_biawgn(code: Code, snr: float, data_key: int, frame_id: int) -> dict:
    """One frame of the virtual BIAWGN channel MD reconciliation creates: Bob's bits
    u, S_B = H u, and Alice's channel LLRs lambda = 2 y snr with y = (1 - 2u) + N(0, 1/snr),
    i.e. lambda ~ N(+-2 snr, 4 snr) (R31)."""
    g = frame_rng(data_key, (1 << 62) | int(frame_id))      # own stream: not the MD frames' draws
    u = g.integers(0, 2, size=code.n, dtype=np.uint8)
    y = (1.0 - 2.0 * u) + g.standard_normal(code.n) / np.sqrt(snr)
    return {"u": u, "llr": (2.0 * snr * y).astype(np.float32), "synd": syndrome_words(code, u),
            "frame_id": frame_id}


def gen_batch_biawgn(code: Code, snr: float, data_key: int, frame_ids) -> dict:
    fr = [gen_frame_biawgn(code, snr, data_key, f) for f in frame_ids]
    return {k: np.stack([f[k] for f in fr]) for k in ("u", "llr", "synd")} | {"frame_ids": np.asarray(list(frame_ids))}

