"""Thin ctypes binding of libmetldpc.so (include/metldpc.h) -- argument marshalling only.

Every ``metldpc_*`` function here forwards to the C ABI of the same name; torch
tensors are passed as ``data_ptr()`` device pointers and the current CUDA stream
as ``cuda_stream``.  There is no CPU fallback: if the shared library is missing
or fails to load, :func:`lib` raises.

Convenience wrappers :class:`Code` and :class:`Decoder` own the handles.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

_PKG = Path(__file__).resolve().parent
# METLDPC_LIB selects an alternative in-tree build (kernel-variant experiments).
LIB_PATH = Path(os.environ["METLDPC_LIB"]) if os.environ.get("METLDPC_LIB") else _PKG / "libmetldpc.so"

OK, EINVAL, EFORMAT, ENOMEM, ECUDA, EUNSUPPORTED = range(6)
RULE_EXACT, RULE_PHI_LUT = 0, 1
CODE_NO_SKIP = 1

_lib = None


class MetLdpcError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {_lib.metldpc_status_string(status).decode()} "
                         f"({_lib.metldpc_last_error().decode()})")


class Config(C.Structure):
    _fields_ = [("rule", C.c_int32), ("max_iter", C.c_int32), ("early_term", C.c_int32),
                ("lanes_per_group", C.c_int32), ("groups_in_flight", C.c_int32), ("lane_refill", C.c_int32),
                ("msg_bits", C.c_int32)]


class CodeInfo(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("edges", C.c_int64), ("iter_edges", C.c_int64),
                ("n_active", C.c_int32), ("n_deg1", C.c_int32), ("max_cn_deg", C.c_int32),
                ("max_vn_deg", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Profile(C.Structure):
    _fields_ = [("launches", C.c_int64), ("cn_launches", C.c_int64), ("vn_launches", C.c_int64),
                ("cn_ms", C.c_double), ("vn_ms", C.c_double), ("cn_lane_iters", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


SYMBOLS = {
    # name: (restype, argtypes)
    "metldpc_code_create": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "metldpc_code_create_ex": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_uint32, C.POINTER(C.c_void_p)]),
    "metldpc_code_load_alist": (C.c_int, [C.c_int32, C.c_char_p, C.POINTER(C.c_void_p)]),
    "metldpc_code_check": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.POINTER(CodeInfo)]),
    "metldpc_code_info": (C.c_int, [C.c_void_p, C.POINTER(CodeInfo)]),
    "metldpc_code_destroy": (None, [C.c_void_p]),
    "metldpc_config_default": (None, [C.POINTER(Config)]),
    "metldpc_decoder_create": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(Config), C.POINTER(C.c_void_p)]),
    "metldpc_decoder_destroy": (None, [C.c_void_p]),
    "metldpc_llr_from_md": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_float, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_size_t]),
    "metldpc_md_alice_llr": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_float, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_size_t]),
    "metldpc_syndrome": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_size_t]),
    "metldpc_decode": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_size_t]),
    "metldpc_decode_host": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                      C.c_void_p, C.c_void_p]),
    "metldpc_decode_md_host": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_float, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "metldpc_batch_counters": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]),
    "metldpc_debug_dump": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "metldpc_debug_step": (C.c_int, [C.c_void_p, C.c_int32, C.c_size_t]),
    "metldpc_phi_table": (C.c_int32, [C.c_int32, C.c_void_p, C.c_int32]),
    "metldpc_set_profiling": (C.c_int, [C.c_void_p, C.c_int32]),
    "metldpc_get_profile": (C.c_int, [C.c_void_p, C.POINTER(Profile)]),
    "metldpc_reset_profile": (C.c_int, [C.c_void_p]),
    "metldpc_status_string": (C.c_char_p, [C.c_int]),
    "metldpc_last_error": (C.c_char_p, []),
}


def lib():
    """Loads libmetldpc.so (fails loudly: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} not built; run `python -m paper_1711_01783_b200.build` "
                               "or __graft_entry__.build()")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SYMBOLS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(status: int, where: str):
    if status != OK:
        raise MetLdpcError(status, where)


def _ptr(t):
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return C.c_void_p(t.data_ptr())
    return t.ctypes.data_as(C.c_void_p)   # numpy (host)


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


# ----------------------------------------------------------------------------- same-name forwards

def metldpc_code_create(device, n, m, num_edges, cn_ptr, edge_vn, vn_ptr, vn_edge):
    h = C.c_void_p()
    _check(lib().metldpc_code_create(device, n, m, num_edges, _ptr(cn_ptr), _ptr(edge_vn), _ptr(vn_ptr),
                                     _ptr(vn_edge), C.byref(h)), "metldpc_code_create")
    return h


def metldpc_code_create_ex(device, n, m, num_edges, cn_ptr, edge_vn, vn_ptr, vn_edge, flags):
    h = C.c_void_p()
    _check(lib().metldpc_code_create_ex(device, n, m, num_edges, _ptr(cn_ptr), _ptr(edge_vn), _ptr(vn_ptr),
                                        _ptr(vn_edge), int(flags), C.byref(h)), "metldpc_code_create_ex")
    return h


def metldpc_code_load_alist(device, path):
    h = C.c_void_p()
    _check(lib().metldpc_code_load_alist(device, str(path).encode(), C.byref(h)), "metldpc_code_load_alist")
    return h


def metldpc_code_check(n, m, num_edges, cn_ptr, edge_vn, vn_ptr, vn_edge):
    info = CodeInfo()
    _check(lib().metldpc_code_check(n, m, num_edges, _ptr(cn_ptr), _ptr(edge_vn), _ptr(vn_ptr), _ptr(vn_edge),
                                    C.byref(info)), "metldpc_code_check")
    return info


def metldpc_code_info(code):
    info = CodeInfo()
    _check(lib().metldpc_code_info(code, C.byref(info)), "metldpc_code_info")
    return info


def metldpc_code_destroy(code):
    lib().metldpc_code_destroy(code)


def metldpc_config_default():
    cfg = Config()
    lib().metldpc_config_default(C.byref(cfg))
    return cfg


def metldpc_decoder_create(code, max_batch, cfg=None):
    h = C.c_void_p()
    _check(lib().metldpc_decoder_create(code, max_batch, C.byref(cfg) if cfg is not None else None, C.byref(h)),
           "metldpc_decoder_create")
    return h


def metldpc_decoder_destroy(dec):
    lib().metldpc_decoder_destroy(dec)


def metldpc_llr_from_md(dec, batch, d, snr, v, xnorm, llr_out, stream=None):
    _check(lib().metldpc_llr_from_md(dec, batch, d, float(snr), _ptr(v), _ptr(xnorm), _ptr(llr_out),
                                     _stream(stream)), "metldpc_llr_from_md")


def metldpc_md_alice_llr(dec, batch, d, snr, x, alpha, llr_out, stream=None):
    _check(lib().metldpc_md_alice_llr(dec, batch, d, float(snr), _ptr(x), _ptr(alpha), _ptr(llr_out),
                                      _stream(stream)), "metldpc_md_alice_llr")


def metldpc_syndrome(dec, batch, bits, synd_out, stream=None):
    _check(lib().metldpc_syndrome(dec, batch, _ptr(bits), _ptr(synd_out), _stream(stream)), "metldpc_syndrome")


def metldpc_decode(dec, batch, llr, syndrome, max_iter, bits_out, iters_out, converged_out, stream=None):
    _check(lib().metldpc_decode(dec, batch, _ptr(llr), _ptr(syndrome), max_iter, _ptr(bits_out), _ptr(iters_out),
                                _ptr(converged_out), _stream(stream)), "metldpc_decode")


def metldpc_decode_host(dec, batch, llr, syndrome, max_iter, bits_out, iters_out, converged_out):
    _check(lib().metldpc_decode_host(dec, batch, _ptr(llr), _ptr(syndrome), max_iter, _ptr(bits_out),
                                     _ptr(iters_out), _ptr(converged_out)), "metldpc_decode_host")


def metldpc_decode_md_host(dec, batch, d, snr, v, xnorm, syndrome, max_iter, bits_out, iters_out, converged_out):
    _check(lib().metldpc_decode_md_host(dec, batch, d, float(snr), _ptr(v), _ptr(xnorm), _ptr(syndrome), max_iter,
                                        _ptr(bits_out), _ptr(iters_out), _ptr(converged_out)),
           "metldpc_decode_md_host")


def metldpc_batch_counters(dec, batch, iters, converged, counters_out, stream=None):
    _check(lib().metldpc_batch_counters(dec, batch, _ptr(iters), _ptr(converged), _ptr(counters_out),
                                        _stream(stream)), "metldpc_batch_counters")


def metldpc_debug_dump(dec, lane, r_out, L_out):
    _check(lib().metldpc_debug_dump(dec, lane, _ptr(r_out), _ptr(L_out)), "metldpc_debug_dump")


def metldpc_debug_step(dec, k, stream=None):
    _check(lib().metldpc_debug_step(dec, k, _stream(stream)), "metldpc_debug_step")


def metldpc_phi_table(rule):
    import numpy as np
    need = lib().metldpc_phi_table(rule, None, 0)
    out = np.zeros(need, np.float32)
    lib().metldpc_phi_table(rule, _ptr(out), need)
    return out


def metldpc_set_profiling(dec, enable):
    _check(lib().metldpc_set_profiling(dec, int(enable)), "metldpc_set_profiling")


def metldpc_get_profile(dec):
    p = Profile()
    _check(lib().metldpc_get_profile(dec, C.byref(p)), "metldpc_get_profile")
    return p


def metldpc_reset_profile(dec):
    _check(lib().metldpc_reset_profile(dec), "metldpc_reset_profile")


# ----------------------------------------------------------------------------- owning wrappers

class Code:
    """H on a device (immutable).  ``code`` is any object with n, m, cn_ptr, edge_vn,
    vn_ptr, vn_edge numpy arrays (e.g. synth.codes.Code)."""

    def __init__(self, code=None, device: int = 0, alist: str | None = None, no_skip: bool = False):
        import numpy as np
        if alist is not None:
            if no_skip:
                raise ValueError("no_skip needs the CSR/CSC arrays (metldpc_code_create_ex)")
            self.h = metldpc_code_load_alist(device, alist)
        else:
            self._keep = [np.ascontiguousarray(code.cn_ptr, np.int64), np.ascontiguousarray(code.edge_vn, np.int32),
                          np.ascontiguousarray(code.vn_ptr, np.int64), np.ascontiguousarray(code.vn_edge, np.int64)]
            self.h = metldpc_code_create_ex(device, code.n, code.m, int(self._keep[1].size), *self._keep,
                                            CODE_NO_SKIP if no_skip else 0)
            del self._keep
        self.info = metldpc_code_info(self.h)
        self.n, self.m = self.info.n, self.info.m
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            metldpc_code_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Decoder:
    """Decoder workspace; ``decode`` takes torch CUDA tensors and returns torch tensors."""

    def __init__(self, code: Code, max_batch: int, rule: int = RULE_EXACT, max_iter: int = 100,
                 early_term: bool = True, lanes_per_group: int = 64, groups_in_flight: int | None = None,
                 lane_refill: bool | None = None, msg_bits: int = 32):
        cfg = metldpc_config_default()
        cfg.msg_bits = msg_bits
        cfg.rule, cfg.max_iter, cfg.early_term, cfg.lanes_per_group = rule, max_iter, int(early_term), lanes_per_group
        if groups_in_flight is not None:
            cfg.groups_in_flight = groups_in_flight
        if lane_refill is not None:
            cfg.lane_refill = int(lane_refill)
        self.cfg = cfg
        self.code = code
        self.max_batch = max_batch
        self.h = metldpc_decoder_create(code.h, max_batch, cfg)

    def llr_from_md(self, v, xnorm, snr: float, d: int = 8, out=None, stream=None):
        import torch
        batch = v.shape[0]
        if out is None:
            out = torch.empty_like(v)
        metldpc_llr_from_md(self.h, batch, d, snr, v, xnorm, out, stream)
        return out

    def md_alice_llr(self, x, alpha, snr: float, d: int = 8, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty_like(x)
        metldpc_md_alice_llr(self.h, x.shape[0], d, snr, x, alpha, out, stream)
        return out

    def syndrome(self, bits, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty((bits.shape[0], (self.code.m + 31) // 32), dtype=torch.int32, device=bits.device)
        metldpc_syndrome(self.h, bits.shape[0], bits, out, stream)
        return out

    def decode(self, llr, syndrome, max_iter: int = 0, stream=None, out=None):
        import torch
        batch = llr.shape[0]
        dev = llr.device
        nw = (self.code.n + 31) // 32
        if out is None:
            out = (torch.empty((batch, nw), dtype=torch.int32, device=dev),
                   torch.empty(batch, dtype=torch.int32, device=dev),
                   torch.empty(batch, dtype=torch.uint8, device=dev))
        bits, iters, conv = out
        metldpc_decode(self.h, batch, llr, syndrome, max_iter, bits, iters, conv, stream)
        return bits, iters, conv

    def decode_host(self, llr, syndrome, max_iter: int = 0, out=None):
        """Host (numpy or pinned torch CPU) buffers in and out."""
        import numpy as np
        batch = llr.shape[0]
        nw = (self.code.n + 31) // 32
        if out is None:
            out = (np.empty((batch, nw), np.uint32), np.empty(batch, np.int32), np.empty(batch, np.uint8))
        metldpc_decode_host(self.h, batch, llr, syndrome, max_iter, *out)
        return out

    def decode_md_host(self, v, xnorm, syndrome, snr: float, d: int = 8, max_iter: int = 0, out=None):
        """Alice's path from HOST MD output: H2D, LLR, decode, D2H inside the library."""
        import numpy as np
        batch = v.shape[0]
        nw = (self.code.n + 31) // 32
        if out is None:
            out = (np.empty((batch, nw), np.uint32), np.empty(batch, np.int32), np.empty(batch, np.uint8))
        metldpc_decode_md_host(self.h, batch, d, snr, v, xnorm, syndrome, max_iter, *out)
        return out

    def counters(self, iters, conv, out, stream=None):
        metldpc_batch_counters(self.h, iters.shape[0], iters, conv, out, stream)
        return out

    def dump(self, lane: int):
        import numpy as np
        r = np.zeros(self.code.info.iter_edges, np.float32)
        L = np.zeros(self.code.info.n_active, np.float32)
        metldpc_debug_dump(self.h, lane, r, L)
        return r, L

    def step(self, k: int = 1, stream=None):
        metldpc_debug_step(self.h, k, stream)

    def set_profiling(self, on: bool):
        metldpc_set_profiling(self.h, on)

    def profile(self) -> dict:
        return metldpc_get_profile(self.h).as_dict()

    def reset_profile(self):
        metldpc_reset_profile(self.h)

    def close(self):
        if getattr(self, "h", None):
            metldpc_decoder_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
