"""C-ABI checks that need no GPU: libgsp.so builds, loads, exports every
symbol include/gsp.h declares, and host-side validation rejects bad
arguments before any launch (gsp.h CONVENTIONS / Errors)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2103_00959_b200 as G
from paper_2103_00959_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gsp.h")


@pytest.fixture(scope="module")
def L():
    _build.build()
    return G.lib()


def declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(gsp_[a-z_0-9]+)\s*\(", txt)))


def test_header_lists_all_exports():
    assert set(declared()) == set(G.EXPORTS)


def test_exports(L):
    nm = subprocess.run(["nm", "-D", "--defined-only", G.LIB_PATH], capture_output=True, text=True).stdout
    syms = set(re.findall(r" T (gsp_\w+)", nm))
    for name in declared():
        assert name in syms, name
        assert hasattr(L, name)


def test_sm100a_cubin(L):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", G.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_and_strings(L):
    assert L.gsp_version() == 2
    assert L.gsp_status_string(0) == b"GSP_OK"
    assert L.gsp_status_string(5) == b"GSP_ERR_ALIAS"


def _csr(n_rows=10, n_cols=10, nnz=20, rp=0x1000, col=0x2000, val=0x3000):
    return G.gsp_csr(n_rows, n_cols, nnz, rp, col, val)


def test_host_validation(L):
    P = ctypes.c_void_p
    s = P(0)
    c = _csr()
    # NULL csr view
    assert L.gsp_spmm(None, P(0x10000), 4, 4, P(0x90000), 4, s) == 1
    # ld < f
    assert L.gsp_spmm(ctypes.byref(c), P(0x10000), 8, 4, P(0x90000), 8, s) == 1
    # negative f
    assert L.gsp_spmm(ctypes.byref(c), P(0x10000), -1, 4, P(0x90000), 4, s) == 1
    # x / y overlap -> ALIAS (checked before any launch)
    assert L.gsp_spmm(ctypes.byref(c), P(0x10000), 4, 4, P(0x10010), 4, s) == 5
    assert b"overlap" in L.gsp_last_error_detail()
    # n >= 2^31 unsupported
    big = _csr(n_rows=1 << 31)
    assert L.gsp_spmm(ctypes.byref(big), P(0x10000), 4, 4, P(0x90000000), 4, s) == 7
    # multi-head: heads * d > ldz
    assert L.gsp_multihead_spmm(ctypes.byref(c), 4, P(0x5000), P(0x10000), 8, 16, P(0x90000), 32, s) == 1
    # softmax heads <= 0
    assert L.gsp_edge_softmax(ctypes.byref(c), 0, P(0x5000), P(0x5000), s) == 1
    # gat: heads * d > ldz
    assert L.gsp_gat_aggregate(ctypes.byref(c), 4, P(0x5000), P(0x6000), 0.2, P(0x10000), 4, 8, P(0x90000), 16,
                               None, None, 0, s) == 1
    # normalize needs values
    c0 = _csr(val=None)
    assert L.gsp_sym_normalize(ctypes.byref(c0), P(0x7000), P(0x8000), None, 0, s) == 1
    # deg_out NULL: a workspace of n_rows doubles is required (nothing launched)
    assert L.gsp_sym_normalize(ctypes.byref(c), P(0x7000), None, None, 0, s) == 6
    assert L.gsp_sym_normalize(ctypes.byref(c), P(0x7000), None, P(0x8000), 79, s) == 6
    assert L.gsp_sym_normalize(ctypes.byref(c), P(0x7000), None, P(0x8004), 80, s) == 6  # misaligned
    # val_out overlapping the degree array
    assert L.gsp_sym_normalize(ctypes.byref(c), P(0x7000), P(0x7010), None, 0, s) == 5
    nb = ctypes.c_size_t(0)
    assert L.gsp_sym_normalize_workspace(ctypes.byref(c), ctypes.byref(nb)) == 0 and nb.value == 80
    # partition parts out of range
    assert L.gsp_partition_rows(ctypes.byref(c), 0, P(0x7000), None, s) == 1
    # slice: bounds must span [0, n)
    hb = (ctypes.c_int64 * 3)(0, 4, 9)
    assert L.gsp_csr_slice(ctypes.byref(c), hb, 2, 0, 5, P(0x7000), P(0x8000), None, s) == 1


def test_host_validation_new_entry_points(L):
    """fp16-storage SpMM and the tensor-core GEMM reject bad arguments on the
    host, before any launch (gsp.h Errors)."""
    P = ctypes.c_void_p
    s = P(0)
    c = _csr()
    # gsp_spmm_f16: ld < f, NULL y, x / y overlap (x counted in 2-byte elements)
    assert L.gsp_spmm_f16(ctypes.byref(c), P(0x10000), 8, 4, P(0x90000), 8, s) == 1
    assert L.gsp_spmm_f16(ctypes.byref(c), P(0x10000), 4, 4, None, 4, s) == 1
    assert L.gsp_spmm_f16(ctypes.byref(c), P(0x10000), 4, 4, P(0x10010), 4, s) == 5
    # gsp_linear: ldw < f_out; x / y overlap
    assert L.gsp_linear(10, 8, P(0x10000), 8, P(0x20000), 2, 4, P(0x90000), 4, None, 0, s) == 1
    assert L.gsp_linear(10, 8, P(0x10000), 8, P(0x20000), 4, 4, P(0x10020), 4, None, 0, s) == 5
    # workspace queries
    n = ctypes.c_size_t(0)
    assert L.gsp_linear_workspace(-1, 4, ctypes.byref(n)) == 1
    assert L.gsp_linear_workspace(602, 128, ctypes.byref(n)) == 0
    assert n.value >= 2 * 128 * 608 * 4  # hi + lo copies of W^T, K padded to the tile
    assert L.gsp_gcn_layer_workspace(1000, 602, 128, ctypes.byref(n)) == 0
    assert n.value >= 1000 * 128 * 4 + 2 * 128 * 608 * 4
    cg = _csr(n_rows=100, n_cols=100, nnz=500)
    assert L.gsp_gat_workspace(ctypes.byref(cg), 8, ctypes.byref(n)) == 0
    # max of the statistics ((m fp64, 1/S fp32, pad) per (row, head)) and the
    # head-major alpha of the staged schedule (nnz rounded up to 32, per head)
    assert n.value == max(100 * 8 * 16, 512 * 8 * 4)


def test_colblock_host_validation(L):
    """Column blocks: workspace query and bound checks on the host, before
    any launch (gsp.h column blocks)."""
    n = ctypes.c_size_t(0)
    c = _csr(n_rows=100, n_cols=100, nnz=500)
    assert L.gsp_csr_colblock_workspace(ctypes.byref(c), 0, ctypes.byref(n)) == 1
    assert L.gsp_csr_colblock_workspace(ctypes.byref(c), 9, ctypes.byref(n)) == 1
    assert L.gsp_csr_colblock_workspace(ctypes.byref(c), 2, ctypes.byref(n)) == 0
    assert n.value >= 2 * 101 * 8 + 500 * 8  # two row_ptr, col + val once
    out = (G.gsp_csr * 2)()
    P = ctypes.c_void_p
    ws = P(0x100000)
    bad = [(0, 60, 99), (1, 60, 100), (0, 60, 40)]  # must span [0, n_cols), nondecreasing
    for b in bad:
        hb = (ctypes.c_int64 * 3)(*b)
        assert L.gsp_csr_colblock(ctypes.byref(c), hb, 2, ws, n.value, out, P(0)) == 1, b
    hb = (ctypes.c_int64 * 3)(0, 50, 100)
    assert L.gsp_csr_colblock(ctypes.byref(c), hb, 2, ws, n.value - 1024, out, P(0)) == 6  # workspace too small
    # gsp_spmm_blocked: no blocks / mismatched shapes
    assert L.gsp_spmm_blocked(None, 1, P(0x1000), 4, 4, P(0x9000), 4, P(0)) == 1
    two = (G.gsp_csr * 2)(_csr(n_rows=100, n_cols=100, nnz=500), _csr(n_rows=99, n_cols=100, nnz=500))
    assert L.gsp_spmm_blocked(two, 2, P(0x1000), 4, 4, P(0x9000), 4, P(0)) == 1


def test_build_workspace_query(L):
    ws = ctypes.c_size_t(0)
    nmax = ctypes.c_int64(0)
    assert L.gsp_coo_to_csr_workspace(100, 1000, 1, 1.0, ctypes.byref(ws), ctypes.byref(nmax)) == 0
    assert nmax.value == 2 * 1000 + 100 and ws.value > 0
    assert L.gsp_coo_to_csr_workspace(100, 1000, 0, 0.0, ctypes.byref(ws), ctypes.byref(nmax)) == 0
    assert nmax.value == 1000
    assert L.gsp_coo_to_csr_workspace(100, 1 << 31, 1, 1.0, ctypes.byref(ws), ctypes.byref(nmax)) == 7
    # host-checked build errors (no launch)
    n = ctypes.c_int64(0)
    assert L.gsp_coo_to_csr(10, 5, None, None, 1, None, 1, 1.0, ctypes.c_void_p(0x100), ctypes.c_void_p(0x200),
                            ctypes.c_void_p(0x300), ctypes.byref(n), ctypes.c_void_p(0x400), 10, None) == 1
    assert L.gsp_coo_to_csr(10, 0, None, None, 1, None, 1, -1.0, ctypes.c_void_p(0x100), ctypes.c_void_p(0x200),
                            ctypes.c_void_p(0x300), ctypes.byref(n), ctypes.c_void_p(0x400), 10, None) == 3
    assert L.gsp_coo_to_csr(10, 0, None, None, 1, None, 1, float("nan"), ctypes.c_void_p(0x100),
                            ctypes.c_void_p(0x200), ctypes.c_void_p(0x300), ctypes.byref(n), ctypes.c_void_p(0x400),
                            10, None) == 4


def test_product_does_not_import_oracle():
    """The product package never imports, links or calls the oracle."""
    pkg = os.path.join(ROOT, "paper_2103_00959_b200")
    pat = re.compile(r"import\s+oracle|from\s+oracle|liboracle|\borc_[a-z]|oracle\.c\b")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not pat.search(txt), f
    nm = subprocess.run(["nm", "-D", G.LIB_PATH], capture_output=True, text=True).stdout
    assert "orc_" not in nm


def test_flags(L):
    """gsp_set_flags: only GSP_VALIDATE is a known bit; the mode is per thread."""
    import threading
    assert L.gsp_get_flags() == 0
    assert L.gsp_set_flags(4) == 1
    assert L.gsp_set_flags(G.GSP_VALIDATE) == 0
    assert L.gsp_get_flags() == G.GSP_VALIDATE
    seen = []
    t = threading.Thread(target=lambda: seen.append(L.gsp_get_flags()))
    t.start()
    t.join()
    assert seen == [0]  # thread-local
    assert L.gsp_set_flags(0) == 0 and L.gsp_get_flags() == 0


def test_gcn_layer_validates_before_enqueue(L):
    """gsp_gcn_layer checks act, sizes, pointers and y / x against the workspace
    before its first enqueue (it used to memset the workspace first)."""
    P = ctypes.c_void_p
    s = P(0)
    c = _csr(n_rows=10, n_cols=10, nnz=20)
    n = ctypes.c_size_t(0)
    assert L.gsp_gcn_layer_workspace(10, 8, 4, ctypes.byref(n)) == 0
    ws = P(0x100000)
    assert L.gsp_gcn_layer(ctypes.byref(c), P(0x10000), 8, 8, P(0x20000), 4, None, 7, P(0x90000), 4, ws, n.value,
                           s) == 1  # bad activation
    assert L.gsp_gcn_layer(ctypes.byref(c), P(0x10000), 8, 4, P(0x20000), 4, None, 1, P(0x90000), 4, ws, n.value,
                           s) == 1  # ldx < f_in
    assert L.gsp_gcn_layer(ctypes.byref(c), P(0x10000), 8, 8, None, 4, None, 1, P(0x90000), 4, ws, n.value,
                           s) == 1  # NULL w
    assert L.gsp_gcn_layer(ctypes.byref(c), P(0x10000), 8, 8, P(0x20000), 4, None, 1, P(0x100010), 4, ws, n.value,
                           s) == 5  # y inside the workspace
    assert L.gsp_gcn_layer(ctypes.byref(c), P(0x10000), 8, 8, P(0x20000), 4, None, 1, P(0x90000), 4, ws, 16,
                           s) == 6  # workspace too small


def test_spmm_ex_slab256_alignment(L):
    """slab_cols 256 (two float4 per lane) is refused unless ldx % 8 == 0 and x
    is 32-byte aligned (the last vector could read past the row)."""
    P = ctypes.c_void_p
    c = _csr()
    o = G.gsp_spmm_opts(256, 0)
    assert L.gsp_spmm_ex(ctypes.byref(c), P(0x10000), 260, 260, P(0x900000), 260, ctypes.byref(o), P(0)) == 1
    assert L.gsp_spmm_ex(ctypes.byref(c), P(0x10010), 256, 264, P(0x900000), 256, ctypes.byref(o), P(0)) == 1
    o2 = G.gsp_spmm_opts(256, 0)
    launches, sc = ctypes.c_int32(0), ctypes.c_int32(0)
    assert L.gsp_spmm_plan_info(ctypes.byref(c), P(0x10000), 300, 304, ctypes.byref(o2), ctypes.byref(launches),
                                ctypes.byref(sc), None) == 0 and sc.value == 256


def test_binding_shape_checks():
    """The binding rejects shape mistakes the C ABI cannot see."""
    import torch
    rp = torch.zeros(4, dtype=torch.int64)
    col = torch.zeros(0, dtype=torch.int32)
    a = G.CSR.__new__(G.CSR)
    a.row_ptr, a.col, a.val, a.n_rows, a.n_cols, a.nnz, a.deg = rp, col, None, 3, 5, 6, None
    x = torch.zeros((4, 8))
    with pytest.raises(ValueError):
        G._rows(x, a.n_cols, "x")
    with pytest.raises(ValueError):
        G._numel(torch.zeros(5), a.nnz, "alpha")
    with pytest.raises(ValueError):
        G._width(x, 9, "x")
