"""ctypes wrapper of oracle/bp_oracle.c (TEST INFRASTRUCTURE; see oracle/__init__.py).

Builds ``liboracle_bp.so`` with gcc on first use if it is missing or older than
the source (``-O2 -ffp-contract=off``, no fast-math: IEEE fp32/fp64 as written).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_DIR = Path(__file__).resolve().parent
_SRC = _DIR / "bp_oracle.c"
_LIB = _DIR / "liboracle_bp.so"

RULE_EXACT = 0
RULE_PHI_LUT = 1
NO_SKIP = 0x100   # variant bit: iterate degree-1 VNs too (Table 1 "without skipping")
MSG16 = 0x200     # fp32 (M3) variant bit: messages stored as rint(2^10 r) 2^-10 (R28/N7)
R_MAX = 30.0

_lib = None


def build(force: bool = False) -> Path:
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(f".{os.getpid()}.tmp")
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-Wall", "-shared", "-fPIC", str(_SRC), "-o", str(tmp), "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(str(build()))
        P = C.c_void_p
        _lib.orc_phi_def.restype = C.c_double
        _lib.orc_phi_def.argtypes = [C.c_double]
        _lib.orc_phi32.restype = C.c_float
        _lib.orc_phi32.argtypes = [C.c_int, C.c_float]
        _lib.orc_phi64.restype = C.c_double
        _lib.orc_phi64.argtypes = [C.c_int, C.c_double]
        _lib.orc_phi_table.restype = C.c_int
        _lib.orc_phi_table.argtypes = [C.c_int, P, C.c_int]
        graph = [C.c_int, C.c_int, P, P, P, P]
        _lib.orc_decode_f32.restype = C.c_int
        _lib.orc_decode_f32.argtypes = [C.c_int] + graph + [P, P, C.c_int, C.c_int, P, P, P, P, P]
        _lib.orc_decode_f64.restype = C.c_int
        _lib.orc_decode_f64.argtypes = [C.c_int] + graph + [P, P, C.c_int, C.c_int, P, P, P, P, P, P]
        _lib.orc_step_f64.restype = C.c_int
        _lib.orc_step_f64.argtypes = [C.c_int] + graph + [P, P, P, P, P, P]
        _lib.orc_graph_sizes.restype = C.c_int
        _lib.orc_graph_sizes.argtypes = [C.c_int] + graph + [P, P]
        _lib.orc_syndrome.restype = None
        _lib.orc_syndrome.argtypes = [C.c_int, C.c_int, P, P, P, P]
        _lib.orc_llr_from_md_f32.restype = None
        _lib.orc_llr_from_md_f32.argtypes = [C.c_int, C.c_int, C.c_float, P, P, P]
        _lib.orc_llr_from_md_f64.restype = None
        _lib.orc_llr_from_md_f64.argtypes = [C.c_int, C.c_int, C.c_double, P, P, P]
        _lib.orc_md_alice_f32.restype = None
        _lib.orc_md_alice_f32.argtypes = [C.c_int, C.c_int, C.c_float, P, P, P]
        _lib.orc_md_table.restype = None
        _lib.orc_md_table.argtypes = [C.c_int, P, P]
        _lib.orc_init()
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _graph(code):
    arrs = (np.ascontiguousarray(code.cn_ptr, np.int64), np.ascontiguousarray(code.edge_vn, np.int32),
            np.ascontiguousarray(code.vn_ptr, np.int64), np.ascontiguousarray(code.vn_edge, np.int64))
    return arrs, [code.n, code.m] + [_p(a) for a in arrs]


def graph_sizes(code, no_skip: bool = False):
    keep, g = _graph(code)
    E_it = np.zeros(1, np.int64)
    n_a = np.zeros(1, np.int32)
    rc = lib().orc_graph_sizes(NO_SKIP if no_skip else 0, *g, _p(E_it), _p(n_a))
    if rc:
        raise ValueError(f"malformed code (rc={rc})")
    return int(E_it[0]), int(n_a[0])


def phi_def(y: float) -> float:
    return lib().orc_phi_def(float(y))


def phi32(rule: int, y: float) -> float:
    return lib().orc_phi32(int(rule), float(y))


def phi64(rule: int, y: float) -> float:
    return lib().orc_phi64(int(rule), float(y))


def phi_table(rule: int) -> np.ndarray:
    need = lib().orc_phi_table(int(rule), None, 0)
    out = np.zeros(need, np.float32)
    lib().orc_phi_table(int(rule), _p(out), need)
    return out


def llr_from_md_f32(v: np.ndarray, xnorm, snr: float, d: int = 8) -> np.ndarray:
    v = np.ascontiguousarray(v, np.float32)
    xn = None if xnorm is None else np.ascontiguousarray(xnorm, np.float32)
    out = np.empty_like(v)
    lib().orc_llr_from_md_f32(v.size, d, float(snr), _p(v), _p(xn), _p(out))
    return out


def llr_from_md_f64(v: np.ndarray, xnorm, snr: float, d: int = 8) -> np.ndarray:
    v = np.ascontiguousarray(v, np.float64)
    xn = None if xnorm is None else np.ascontiguousarray(xnorm, np.float64)
    out = np.empty_like(v)
    lib().orc_llr_from_md_f64(v.size, d, float(snr), _p(v), _p(xn), _p(out))
    return out


def syndrome(code, bits: np.ndarray) -> np.ndarray:
    keep, g = _graph(code)
    c = np.ascontiguousarray(bits, np.uint8)
    s = np.zeros(code.m, np.uint8)
    lib().orc_syndrome(code.n, code.m, g[2], g[3], _p(c), _p(s))
    return s


def decode(code, llr: np.ndarray, synd_words: np.ndarray, max_iter: int, early_term: bool = True,
           rule: int = RULE_EXACT, prec: int = 32, trace: bool = False, posterior: bool = False,
           no_skip: bool = False, msg16: bool = False):
    """Decode ONE frame.  prec=32 -> M3 (fp32 replay), prec=64 -> M2 (fp64 definition).
    no_skip iterates degree-1 VNs too (Table 1 "without skipping", R26).
    msg16 (M3 only) stores the messages in 16 bits, rint(2^10 r) 2^-10 (R28/N7);
    r_trace then holds the stored messages.

    Returns dict(bits uint8[n], iters, converged, [r_trace, L_trace], [post]).
    """
    keep, g = _graph(code)
    s = np.ascontiguousarray(synd_words, np.uint32)
    bits = np.zeros(code.n, np.uint8)
    it = np.zeros(1, np.int32)
    cv = np.zeros(1, np.uint8)
    out = {}
    rt = Lt = None
    if trace:
        E_it, n_a = graph_sizes(code, no_skip)
    if no_skip:
        rule = rule | NO_SKIP
    if msg16:
        if prec != 32:
            raise ValueError("msg16 is an fp32 (M3) storage variant")
        rule = rule | MSG16
    if prec == 32:
        lam = np.ascontiguousarray(llr, np.float32)
        if trace:
            rt = np.zeros((max_iter, E_it), np.float32)
            Lt = np.zeros((max_iter, n_a), np.float32)
        rc = lib().orc_decode_f32(rule, *g, _p(lam), _p(s), max_iter, int(early_term),
                                  _p(bits), _p(it), _p(cv), _p(rt), _p(Lt))
    elif prec == 64:
        lam = np.ascontiguousarray(llr, np.float64)
        if trace:
            rt = np.zeros((max_iter, E_it), np.float64)
            Lt = np.zeros((max_iter, n_a), np.float64)
        post = np.zeros(code.n, np.float64) if posterior else None
        rc = lib().orc_decode_f64(rule, *g, _p(lam), _p(s), max_iter, int(early_term),
                                  _p(bits), _p(it), _p(cv), _p(rt), _p(Lt), _p(post))
        if posterior:
            out["post"] = post
    else:
        raise ValueError("prec must be 32 or 64")
    if rc:
        raise ValueError(f"malformed code (rc={rc})")
    out.update(bits=bits, iters=int(it[0]), converged=bool(cv[0]))
    if trace:
        k = max(int(it[0]), 0)
        out["r_trace"], out["L_trace"] = rt[:k], Lt[:k]
    return out


def step64(code, llr, synd_words, r_in, L_in, rule: int = RULE_EXACT, no_skip: bool = False):
    """One fp64 iteration from (r^{l-1}, L^{l-1}) -> (r^l, L^l)."""
    keep, g = _graph(code)
    E_it, n_a = graph_sizes(code, no_skip)
    if no_skip:
        rule = rule | NO_SKIP
    lam = np.ascontiguousarray(llr, np.float64)
    s = np.ascontiguousarray(synd_words, np.uint32)
    ri = np.ascontiguousarray(r_in, np.float64)
    Li = np.ascontiguousarray(L_in, np.float64)
    ro = np.zeros(E_it, np.float64)
    Lo = np.zeros(n_a, np.float64)
    rc = lib().orc_step_f64(rule, *g, _p(lam), _p(s), _p(ri), _p(Li), _p(ro), _p(Lo))
    if rc:
        raise ValueError(f"malformed code (rc={rc})")
    return ro, Lo


def md_alice_f32(x: np.ndarray, alpha: np.ndarray, snr: float, d: int = 8) -> np.ndarray:
    """DESIGN.md N6: lambda = c * (alpha x) per d-block (octonion product in a fixed fmaf order)."""
    x = np.ascontiguousarray(x, np.float32)
    a = np.ascontiguousarray(alpha, np.float32)
    out = np.empty_like(x)
    lib().orc_md_alice_f32(x.size, d, float(snr), _p(x), _p(a), _p(out))
    return out


def md_table(d: int):
    k = np.zeros(d * d, np.int32)
    s = np.zeros(d * d, np.int32)
    lib().orc_md_table(d, _p(k), _p(s))
    return k.reshape(d, d), s.reshape(d, d)
