"""GPU (torch) generator of CV-QKD frames for large statistical runs (C5 FER sweeps).

Same model as synth/frames.py -- X ~ N(0,1), Z ~ N(0, 1/snr), Y = X + Z, Bob's bits U,
8-D MD rotation alpha = u~ * conj(y^) (Cayley-Dickson product) -- drawn with torch's
Philox generator on the device, seeded by (data key, batch index).  Input generation only:
Bob's syndrome, Alice's LLRs and the decoding run in the library (metldpc_syndrome,
metldpc_md_alice_llr, metldpc_decode).  Frames are NOT bit-identical to synth/frames.py
(different generator); parity tests use synth/frames.py.
"""
from __future__ import annotations

import torch


def _conj(a):
    out = -a
    out[..., 0] = a[..., 0]
    return out


def cd_mul(a, b):
    d = a.shape[-1]
    if d == 1:
        return a * b
    h = d // 2
    a1, a2 = a[..., :h], a[..., h:]
    b1, b2 = b[..., :h], b[..., h:]
    return torch.cat([cd_mul(a1, b1) - cd_mul(_conj(b2), a2), cd_mul(b2, a1) + cd_mul(a2, _conj(b1))], dim=-1)


def pack_bits(u: torch.Tensor) -> torch.Tensor:
    """uint8 [batch][n] (n % 32 == 0) -> int32 [batch][n/32], LSB-first."""
    b, n = u.shape
    w = u.view(b, n // 32, 32).to(torch.int64) << torch.arange(32, device=u.device, dtype=torch.int64)
    return w.sum(-1).to(torch.uint32).view(torch.int32) if hasattr(torch, "uint32") else \
        (w.sum(-1) - ((w.sum(-1) >> 31) << 32)).to(torch.int32)


def gen_batch(n: int, batch: int, snr: float, key: int, index: int, d: int = 8, device="cuda"):
    """Returns x, alpha (fp32 [batch][n]) and Bob's bits u (uint8 [batch][n])."""
    g = torch.Generator(device=device)
    g.manual_seed((int(key) << 32) ^ (int(index) * 0x9E3779B1) ^ int(round(snr * 1e6)))
    x = torch.randn(batch, n, generator=g, device=device, dtype=torch.float64)
    z = torch.randn(batch, n, generator=g, device=device, dtype=torch.float64) / snr ** 0.5
    u = torch.randint(0, 2, (batch, n), generator=g, device=device, dtype=torch.uint8)
    y = (x + z).view(batch, n // d, d)
    yh = y / torch.linalg.vector_norm(y, dim=-1, keepdim=True)
    ut = (1.0 - 2.0 * u.view(batch, n // d, d).to(torch.float64)) / d ** 0.5
    alpha = cd_mul(ut, _conj(yh)).reshape(batch, n)
    return x.to(torch.float32).contiguous(), alpha.to(torch.float32).contiguous(), u


def gen_batch_biawgn(n: int, batch: int, snr: float, key: int, index: int, device="cuda"):
    """Virtual BIAWGN channel (R31): Bob's bits u (uint8 [batch][n]) and Alice's
    LLRs lambda = 2 snr y, y = (1 - 2u) + N(0, 1/snr) (fp32 [batch][n])."""
    g = torch.Generator(device=device)
    g.manual_seed((int(key) << 32) ^ (int(index) * 0x9E3779B1) ^ int(round(snr * 1e6)) ^ 0x5BD1E995)
    u = torch.randint(0, 2, (batch, n), generator=g, device=device, dtype=torch.uint8)
    y = (1.0 - 2.0 * u.to(torch.float64)) + torch.randn(batch, n, generator=g, device=device,
                                                        dtype=torch.float64) / snr ** 0.5
    return (2.0 * snr * y).to(torch.float32).contiguous(), u

