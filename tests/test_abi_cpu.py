"""-m "not gpu": the C-ABI library loads and exports every symbol include/knnjoin.h declares; host-only
size queries and argument errors behave as documented (no device access)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "knnjoin.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(knnjoin_[a-z_]+)\s*\(", src)))


def test_header_declares_the_survey_entry_points():
    names = _declared()
    for n in ["knnjoin_build_index", "knnjoin_query", "knnjoin_merge", "knnjoin_validate_csr", "knnjoin_index_bytes",
              "knnjoin_build_workspace_bytes", "knnjoin_query_workspace_bytes", "knnjoin_free_index",
              "knnjoin_last_error", "knnjoin_index_stats"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    import paper_1011_2807_b200 as kj
    lib = ctypes.CDLL(kj.library_path())
    for n in _declared():
        assert hasattr(lib, n), n
    assert "sm_100a" in kj.knnjoin_version()


def test_index_bytes_host_only():
    import paper_1011_2807_b200._binding as b
    L = b._lib
    S = b._CSR(100_000, 4_000_000, 0, 0, 0, b.BINARY)
    opt = b._Options(8192, 0, 0.0, 0.0, 0)
    n = L.knnjoin_index_bytes(ctypes.byref(S), 10_000, ctypes.byref(opt))
    nt = (100_000 + 8191) // 8192
    n_off = 10_000 * (nt + 1) + 1
    cap = 4_000_000 // 8 + min(4_000_000, 10_000 * nt) + 1
    al = lambda x: (x + 255) // 256 * 256
    at = al(4 * n_off)          # off
    at = al(at + 4 * 10_000)    # df
    at = al(at + 4 * 10_000)    # head_slot
    at = al(at + 4 * 33)        # head_feat + n_head
    at = al(at + 4 * nt * 8192)  # head_cols
    at = al(at + 16 * cap)       # ids
    assert n == al(at + 4)       # wmax
    # FP32 S: 8 fp32 weights per 16-byte unit of ids
    Sf = b._CSR(100_000, 4_000_000, 0, 0, 0, b.FP32)
    nf = L.knnjoin_index_bytes(ctypes.byref(Sf), 10_000, ctypes.byref(opt))
    assert nf == al(at + 32 * cap) + 256


@pytest.mark.parametrize("d,tile,dtype,msg", [(0, 8192, 0, "d must be"), (100, 1000, 0, "tile"), (100, 8192, 7, "dtype")])
def test_build_argument_errors(d, tile, dtype, msg):
    import paper_1011_2807_b200._binding as b
    L = b._lib
    S = b._CSR(10, 20, 0, 0, 0, dtype)
    opt = b._Options(tile, 0, 0.0, 0.0, 0)
    assert L.knnjoin_index_bytes(ctypes.byref(S), d, ctypes.byref(opt)) == 0
    assert msg in b.knnjoin_last_error()


def test_prune_index_bytes_and_argument_errors():
    """prune = 1 reserves S's forward rows (+ per-feature max weights for INT8 S); bad prune / alpha fail."""
    import paper_1011_2807_b200._binding as b
    L = b._lib
    al = lambda x: (x + 255) // 256 * 256
    for dt, extra in ((b.BINARY, lambda n, z, d: al(8 * (n + 1)) + al(4 * z)),
                      (b.INT8, lambda n, z, d: al(8 * (n + 1)) + al(4 * z) + al(z) + al(4 * d))):
        S = b._CSR(50_000, 1_000_000, 0, 0, 0, dt)
        base = L.knnjoin_index_bytes(ctypes.byref(S), 10_000, ctypes.byref(b._Options(8192, 0, 0.0, 0.0, 0)))
        pr = L.knnjoin_index_bytes(ctypes.byref(S), 10_000, ctypes.byref(b._Options(8192, 1, 0.5, 0.0, 0)))
        assert base > 0 and pr == base + extra(50_000, 1_000_000, 10_000)
    S = b._CSR(10, 20, 0, 0, 0, b.BINARY)
    for opt, msg in ((b._Options(8192, 2, 0.0, 0.0, 0), "prune"), (b._Options(8192, 1, 1.5, 0.0, 0), "alpha"),
                     (b._Options(8192, 0, 0.5, 0.0, 0), "alpha")):
        assert L.knnjoin_index_bytes(ctypes.byref(S), 100, ctypes.byref(opt)) == 0
        assert msg in b.knnjoin_last_error()
    # FP32 S has no 32-bit path: pruned (a6) / residual (f1) indexes need BINARY or INT8 S
    Sf = b._CSR(10, 20, 0, 0, 0, b.FP32)
    assert L.knnjoin_index_bytes(ctypes.byref(Sf), 100, ctypes.byref(b._Options(8192, 1, 0.5, 0.0, 0))) == 0
    assert "FP32 S" in b.knnjoin_last_error()


def test_ctypes_structs_match_the_c_header(tmp_path):
    """The binding's ctypes structures have the C header's sizes and field offsets (compiled with gcc)."""
    import shutil
    import subprocess
    import paper_1011_2807_b200._binding as b
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    structs = {"knnjoin_csr": b._CSR, "knnjoin_options": b._Options, "knnjoin_query_options": b._QueryOptions,
               "knnjoin_index_info": b._IndexInfo, "knnjoin_merge_options": b._MergeOptions}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "knnjoin.h"', "int main(void) {"]
    for cname, cls in structs.items():
        lines.append(f'  printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'  printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call([cc, "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = dict(l.split() for l in subprocess.check_output([str(exe)], text=True).splitlines())
    for cname, cls in structs.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for f, _ in cls._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(cls, f).offset, f"{cname}.{f}"


def test_iiib_host_sizes_and_errors():
    """f1 building blocks: host-only size queries and argument errors (no device access)."""
    import paper_1011_2807_b200._binding as b
    L = b._lib
    R = b._CSR(1000, 40_000, 0, 0, 0, b.FP32)
    S = b._CSR(10_000, 400_000, 0, 0, 0, b.BINARY)
    # (the profile / split sizes include CUB scratch, whose size query needs a device: GPU tests cover them)
    assert L.knnjoin_iiib_profile_bytes(ctypes.byref(R), 0) == 0 and "d <= 0" in b.knnjoin_last_error()
    assert L.knnjoin_iiib_threshold_workspace_bytes(ctypes.byref(R)) >= 16 * 1000
    # NULL profile / threshold -> ERR_ARG before any device work
    st = L.knnjoin_iiib_split(ctypes.byref(S), 10_000, None, None, 1, None, None, None, None, None, None, None, 0, None)
    assert st == 1 and "iiib_split" in b.knnjoin_last_error()
    # forward rows need prune = 1 and S's row count
    F = b._CSR(10_000, 100, 0, 0, 0, b.BINARY)
    opt = b._Options(8192, 0, 0.0, 0.0, 0, ctypes.addressof(F))
    assert L.knnjoin_index_bytes(ctypes.byref(S), 10_000, ctypes.byref(opt)) == 0
    assert "forward" in b.knnjoin_last_error()
    F2 = b._CSR(9_999, 100, 0, 0, 0, b.BINARY)
    opt = b._Options(8192, 1, 0.0, 0.0, 0, ctypes.addressof(F2))
    assert L.knnjoin_index_bytes(ctypes.byref(S), 10_000, ctypes.byref(opt)) == 0
    # with a matching forward CSR the storage holds ITS rows (100 entries), not S's
    opt = b._Options(8192, 1, 0.0, 0.0, 0, ctypes.addressof(F))
    a = L.knnjoin_index_bytes(ctypes.byref(S), 10_000, ctypes.byref(opt))
    base = L.knnjoin_index_bytes(ctypes.byref(S), 10_000, ctypes.byref(b._Options(8192, 0, 0.0, 0.0, 0, None)))
    al = lambda x: (x + 255) // 256 * 256
    assert a == base + al(8 * 10_001) + al(4 * 100)
