"""CPU tests of the C-ABI library: it loads, exports every declared symbol, and its
host-side logic (validation, layout statistics, alist parsing, phi tables) is
right -- no compute call needs a GPU here."""
import ctypes as C
import re
import subprocess

import numpy as np
import pytest

from paper_1711_01783_b200 import binding as B
from synth.codes import Code, from_dense, make_met_code, write_alist


@pytest.fixture(scope="module")
def lib(root):
    from paper_1711_01783_b200.build import build
    build()
    return B.lib()


def declared_symbols(root):
    hdr = (root / "include" / "metldpc.h").read_text()
    decl = r"^(?:const char\*|void|int32_t|metldpc_status)\s+(metldpc_\w+)\s*\("
    return sorted(set(re.findall(decl, hdr, flags=re.M)))


def test_exports_every_declared_symbol(lib, root):
    names = declared_symbols(root)
    assert len(names) >= 18
    out = subprocess.run(["nm", "-D", "--defined-only", str(B.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (metldpc_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert hasattr(lib, n)
    assert set(B.SYMBOLS) == set(names)


def test_status_strings(lib):
    assert B.lib().metldpc_status_string(0) == b"ok"
    assert B.lib().metldpc_status_string(2) == b"malformed parity-check matrix"


def _check(code: Code):
    return B.metldpc_code_check(code.n, code.m, code.num_edges, np.ascontiguousarray(code.cn_ptr, np.int64),
                                np.ascontiguousarray(code.edge_vn, np.int32),
                                np.ascontiguousarray(code.vn_ptr, np.int64), np.ascontiguousarray(code.vn_edge, np.int64))


def test_layout_stats_spec_example(lib):
    """H = [[1,1,0],[0,1,1]] -> VN degrees (1,2,1), 2 iterating edges."""
    info = _check(from_dense(np.array([[1, 1, 0], [0, 1, 1]])))
    assert (info.n, info.m, info.edges, info.iter_edges, info.n_active, info.n_deg1) == (3, 2, 4, 2, 1, 2)


def test_layout_stats_table1(lib):
    """rate-0.1 n=10^6 stand-in -> 3,767,500 edges, 2,892,500 iterating edges."""
    info = _check(make_met_code("r0.1", 10 ** 6))
    assert (info.edges, info.iter_edges, info.n_active, info.n_deg1, info.m) == (3767500, 2892500, 125000, 875000, 900000)


def _corrupt(code: Code, what: str) -> Code:
    c = Code(code.n, code.m, code.cn_ptr.copy(), code.edge_vn.copy(), code.vn_ptr.copy(), code.vn_edge.copy())
    if what == "vn_range":
        c.edge_vn[3] = c.n + 4
    elif what == "dup":
        # make row 0 list its first VN twice
        c.edge_vn[1] = c.edge_vn[0]
    elif what == "csc_perm":
        c.vn_edge[0] = c.vn_edge[1]
    elif what == "csc_mismatch":
        c.vn_edge[[0, -1]] = c.vn_edge[[-1, 0]]
    elif what == "cn_ptr":
        c.cn_ptr[-1] += 1
    return c


@pytest.mark.parametrize("what", ["vn_range", "dup", "csc_perm", "csc_mismatch", "cn_ptr"])
def test_malformed_code_rejected(lib, code_c1, what):
    with pytest.raises(B.MetLdpcError) as ei:
        _check(_corrupt(code_c1, what))
    assert ei.value.status == B.EFORMAT


def test_degree0_vn_rejected(lib):
    h = np.array([[1, 1, 0], [0, 1, 0]])
    with pytest.raises(B.MetLdpcError) as ei:
        _check(from_dense(h))
    assert ei.value.status == B.EFORMAT and "degree 0" in str(ei.value)


def test_cn_degree_limit(lib):
    h = np.ones((1, 33), np.uint8)
    with pytest.raises(B.MetLdpcError) as ei:
        _check(from_dense(h))
    assert ei.value.status == B.EUNSUPPORTED


@pytest.mark.parametrize("rule", [B.RULE_EXACT, B.RULE_PHI_LUT])
def test_phi_table_equals_oracle(lib, rule):
    """DESIGN.md R7/N2: the library and the oracle build the fp32 table independently;
    they must agree entry by entry (bitwise), including PHI_TOP."""
    from oracle import bp
    lt = B.metldpc_phi_table(rule)
    ot = bp.phi_table(rule)
    assert lt.size == ot.size + 1
    assert np.array_equal(lt[:-1].view(np.uint32), ot.view(np.uint32))
    assert np.float32(lt[-1]) == np.float32(bp.phi32(rule, 0.0))


def test_alist_errors_name_the_line(lib, tmp_path):
    p = tmp_path / "bad.alist"
    p.write_text("3 2\n2 2\n1 2 1\n2 2\n1\n1 2\n2\n1 2\n2 4\n")
    h = C.c_void_p()
    st = B.lib().metldpc_code_load_alist(0, str(p).encode(), C.byref(h))
    assert st == B.EFORMAT
    assert b"alist line 9" in B.lib().metldpc_last_error() and b"VN index 4" in B.lib().metldpc_last_error()


def test_decoder_needs_gpu(lib, code_c1):
    """Without a CUDA device code creation fails loudly (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(B.MetLdpcError) as ei:
        B.Code(code_c1)
    assert ei.value.status == B.EUNSUPPORTED


def test_struct_layouts_match_the_header(lib, root, tmp_path):
    """The ctypes mirrors of metldpc_config_t / metldpc_code_info_t / metldpc_profile_t have
    the C sizes and field offsets (a gcc probe compiled against include/metldpc.h), and
    metldpc_config_default fills the documented defaults."""
    probe = tmp_path / "probe.c"
    fields = {"metldpc_config_t": [f for f, _ in B.Config._fields_],
              "metldpc_code_info_t": [f for f, _ in B.CodeInfo._fields_],
              "metldpc_profile_t": [f for f, _ in B.Profile._fields_]}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "metldpc.h"', "int main(void) {"]
    for t, fs in fields.items():
        lines.append(f'printf("{t} %zu\\n", sizeof({t}));')
        for f in fs:
            lines.append(f'printf("{t}.{f} %zu\\n", offsetof({t}, {f}));')
    lines.append("return 0; }")
    probe.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.check_call(["gcc", "-std=c11", f"-I{root / 'include'}", str(probe), "-o", str(exe)])
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    for t, cls in (("metldpc_config_t", B.Config), ("metldpc_code_info_t", B.CodeInfo), ("metldpc_profile_t", B.Profile)):
        assert int(got[t]) == C.sizeof(cls), t
        for f in fields[t]:
            assert int(got[f"{t}.{f}"]) == getattr(cls, f).offset, (t, f)
    cfg = B.metldpc_config_default()
    assert (cfg.rule, cfg.max_iter, cfg.early_term, cfg.lanes_per_group, cfg.groups_in_flight, cfg.lane_refill) == \
        (B.RULE_EXACT, 100, 1, 64, 1, 1)
