"""paper_2103_00959_b200 -- B200-native (sm_100a) sparse GNN operators after
CogDL (arXiv 2103.00959, §4 "Efficiency of CogDL").

This module is the thin Python binding of the C ABI in include/gsp.h: every
function below has the name of the C entry point it calls and does argument
marshalling only (torch tensors -> device pointers + sizes + the current
stream).  Every step of the path runs in libgsp.so's CUDA kernels; there is
no CPU fallback -- if libgsp.so is missing the call raises.

PyTorch is used for device memory, streams and process groups only.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# GSP_LIB selects a tuning variant of the same library (tools/variants.sh); default: the in-tree build
LIB_PATH = os.environ.get("GSP_LIB") or os.path.join(_HERE, "libgsp.so")

GSP_OK = 0
GSP_UNDIRECTED = 1
GSP_VALIDATE = 2
GSP_I32, GSP_I64 = 0, 1
STATUS = {0: "GSP_OK", 1: "GSP_ERR_INVALID_ARG", 2: "GSP_ERR_INDEX_RANGE", 3: "GSP_ERR_NEGATIVE_WEIGHT",
          4: "GSP_ERR_NONFINITE", 5: "GSP_ERR_ALIAS", 6: "GSP_ERR_WORKSPACE", 7: "GSP_ERR_UNSUPPORTED",
          8: "GSP_ERR_CUDA"}

# every symbol include/gsp.h declares
EXPORTS = ("gsp_coo_to_csr_workspace", "gsp_coo_to_csr", "gsp_sym_normalize", "gsp_spmm", "gsp_spmm_f16", "gsp_spmm_ex",
           "gsp_edge_softmax", "gsp_multihead_spmm", "gsp_attn_project", "gsp_gat_workspace", "gsp_gat_aggregate",
           "gsp_partition_rows", "gsp_csr_slice", "gsp_status_string", "gsp_last_error_detail", "gsp_version",
           "gsp_csr_colblock_workspace", "gsp_csr_colblock", "gsp_spmm_blocked",
           "gsp_spmm_plan_info", "gsp_gspmm", "gsp_spmm_accumulate", "gsp_set_flags", "gsp_get_flags",
           "gsp_sym_normalize_workspace",
           "gsp_propagate_workspace", "gsp_propagate", "gsp_csr_transpose_workspace", "gsp_csr_transpose",
           "gsp_sddmm", "gsp_edge_softmax_backward", "gsp_gat_backward_workspace", "gsp_gat_aggregate_backward",
           "gsp_attn_project_backward_workspace", "gsp_attn_project_backward", "gsp_linear_workspace", "gsp_linear",
           "gsp_spmm_bias_act",
           "gsp_gcn_layer_workspace", "gsp_gcn_layer", "gsp_gat_aggregate_bias_act")


class GspError(RuntimeError):
    def __init__(self, status: int, fn: str, detail: str):
        super().__init__(f"{fn}: {STATUS.get(status, status)}: {detail}")
        self.status = status


class gsp_csr(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("n_cols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p), ("val", ctypes.c_void_p)]


class gsp_spmm_opts(ctypes.Structure):
    _fields_ = [("slab_cols", ctypes.c_int32), ("block_nnz", ctypes.c_int32), ("reserved", ctypes.c_int32 * 6)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libgsp.so (raises if it has not been built -- never falls back)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2103_00959_b200._build` "
                               "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        P, I, I32, F, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float, ctypes.c_double
        CP = ctypes.POINTER(gsp_csr)
        sig = {
            "gsp_coo_to_csr_workspace": [I, I, ctypes.c_uint32, F, ctypes.POINTER(ctypes.c_size_t),
                                         ctypes.POINTER(ctypes.c_int64)],
            "gsp_coo_to_csr": [I, I, P, P, ctypes.c_int, P, ctypes.c_uint32, F, P, P, P,
                               ctypes.POINTER(ctypes.c_int64), P, ctypes.c_size_t, P],
            "gsp_sym_normalize": [CP, P, P, P, ctypes.c_size_t, P],
            "gsp_sym_normalize_workspace": [CP, ctypes.POINTER(ctypes.c_size_t)],
            "gsp_spmm": [CP, P, I, I, P, I, P],
            "gsp_spmm_f16": [CP, P, I, I, P, I, P],
            "gsp_spmm_ex": [CP, P, I, I, P, I, ctypes.POINTER(gsp_spmm_opts), P],
            "gsp_gspmm": [CP, ctypes.c_int, P, I, I, P, I, P],
            "gsp_spmm_accumulate": [CP, P, I, I, P, I, P, I, F, P, I, F, P],
            "gsp_propagate_workspace": [CP, I, I, ctypes.POINTER(ctypes.c_size_t)],
            "gsp_propagate": [CP, P, I, I, I, P, P, I, P, ctypes.c_size_t, P],
            "gsp_csr_transpose_workspace": [CP, ctypes.POINTER(ctypes.c_size_t)],
            "gsp_csr_transpose": [CP, P, P, P, P, ctypes.c_size_t, P],
            "gsp_sddmm": [CP, I32, P, I, I, P, I, P, P],
            "gsp_edge_softmax_backward": [CP, I32, P, P, P, P],
            "gsp_gat_backward_workspace": [CP, I32, ctypes.POINTER(ctypes.c_size_t)],
            "gsp_gat_aggregate_backward": [CP, CP, P, I32, P, P, D, P, I, I, P, I, P, I, P, P, P, ctypes.c_size_t, P],
            "gsp_attn_project_backward_workspace": [I, I32, I, ctypes.POINTER(ctypes.c_size_t)],
            "gsp_attn_project_backward": [I, I32, I, P, I, P, P, P, P, P, I, P, P, P, ctypes.c_size_t, P],
            "gsp_linear_workspace": [I, I, ctypes.POINTER(ctypes.c_size_t)],
            "gsp_linear": [I, I, P, I, P, I, I, P, I, P, ctypes.c_size_t, P],
            "gsp_spmm_bias_act": [CP, P, I, I, P, ctypes.c_int, P, I, P],
            "gsp_gcn_layer_workspace": [I, I, I, ctypes.POINTER(ctypes.c_size_t)],
            "gsp_gcn_layer": [CP, P, I, I, P, I, P, ctypes.c_int, P, I, P, ctypes.c_size_t, P],
            "gsp_gat_aggregate_bias_act": [CP, I32, P, P, D, P, I, I, P, ctypes.c_int, P, I, P, ctypes.c_size_t, P],
            "gsp_spmm_plan_info": [CP, P, I, I, ctypes.POINTER(gsp_spmm_opts), ctypes.POINTER(ctypes.c_int32),
                                   ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)],
            "gsp_edge_softmax": [CP, I32, P, P, P],
            "gsp_multihead_spmm": [CP, I32, P, P, I, I, P, I, P],
            "gsp_attn_project": [I, I32, I, P, I, P, P, P, P, P],
            "gsp_gat_workspace": [CP, I32, ctypes.POINTER(ctypes.c_size_t)],
            "gsp_gat_aggregate": [CP, I32, P, P, D, P, I, I, P, I, P, P, ctypes.c_size_t, P],
            "gsp_partition_rows": [CP, I32, P, P, P],
            "gsp_csr_slice": [CP, P, I32, I32, I, P, P, P, P],
            "gsp_csr_colblock_workspace": [CP, I32, ctypes.POINTER(ctypes.c_size_t)],
            "gsp_csr_colblock": [CP, P, I32, P, ctypes.c_size_t, CP, P],
            "gsp_spmm_blocked": [CP, I32, P, I, I, P, I, P],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.gsp_status_string.argtypes = [ctypes.c_int]
        L.gsp_status_string.restype = ctypes.c_char_p
        L.gsp_last_error_detail.argtypes = []
        L.gsp_last_error_detail.restype = ctypes.c_char_p
        L.gsp_set_flags.argtypes = [ctypes.c_uint32]
        L.gsp_set_flags.restype = ctypes.c_int
        L.gsp_get_flags.argtypes = []
        L.gsp_get_flags.restype = ctypes.c_uint32
        L.gsp_version.argtypes = []
        L.gsp_version.restype = ctypes.c_int
        _lib = L
    return _lib


def _check(st: int, fn: str):
    if st != GSP_OK:
        raise GspError(st, fn, lib().gsp_last_error_detail().decode())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _need(t: torch.Tensor, dtype, name: str):
    if not isinstance(t, torch.Tensor) or t.dtype != dtype or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA {dtype} tensor")


def _vec(t: torch.Tensor, dtype, name: str) -> torch.Tensor:
    _need(t, dtype, name)
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _mat(t: torch.Tensor, name: str):
    """(tensor, ld) of a row-major fp32 matrix with unit column stride."""
    _need(t, torch.float32, name)
    if t.dim() != 2 or (t.shape[1] > 1 and t.stride(1) != 1):
        raise ValueError(f"{name} must be 2-D with unit column stride")
    ld = t.stride(0) if t.shape[0] > 1 else max(t.shape[1], t.stride(0))
    return t, ld


# Feature rows are laid out on whole 128-byte L2 lines: a row-slab the SpMM
# gathers then fills whole lines, so one slab of X occupies exactly its bytes
# of L2 (C4: 5.39 -> 4.6 ms for ld 604 -> 608, tools/ld_probe.py).
FEATURE_ALIGN_BYTES = 128


def feature_ld(f: int, dtype=torch.float32) -> int:
    """Row stride (elements) of a feature matrix of width f in the library's
    layout: rows of >= 128 bytes padded to whole 128-byte lines; narrower rows
    to the next power of two of bytes (>= 16), so rows tile lines exactly."""
    es = torch.empty((), dtype=dtype).element_size()
    b = max(int(f), 1) * es
    if b >= FEATURE_ALIGN_BYTES:
        b = (b + FEATURE_ALIGN_BYTES - 1) // FEATURE_ALIGN_BYTES * FEATURE_ALIGN_BYTES
    else:
        p = 16
        while p < b:
            p *= 2
        b = p
    return b // es


def empty_features(n: int, f: int, device, dtype=torch.float32) -> torch.Tensor:
    """[n, f] view of an [n, feature_ld(f)] buffer (128-byte aligned rows, the
    padding columns zeroed: kernels may read them, gsp.h)."""
    ld = feature_ld(f, dtype)
    buf = torch.empty((n, ld), dtype=dtype, device=device)
    if ld > f:
        buf[:, f:].zero_()
    return buf[:, :f]


def _rows(t: torch.Tensor, n: int, name: str):
    """The C ABI cannot see tensor extents: catch caller shape mistakes here."""
    if t.shape[0] < n:
        raise ValueError(f"{name} has {t.shape[0]} rows, needs >= {n}")


def _numel(t: torch.Tensor, n: int, name: str):
    if t.numel() < n:
        raise ValueError(f"{name} has {t.numel()} elements, needs >= {n}")


def _width(t: torch.Tensor, f: int, name: str):
    if t.dim() != 2 or t.shape[1] < f:
        raise ValueError(f"{name} must be 2-D with >= {f} columns, got {tuple(t.shape)}")


class CSR:
    """Device CSR held in torch tensors; .view() is the borrowed gsp_csr."""

    def __init__(self, row_ptr: torch.Tensor, col: torch.Tensor, val: Optional[torch.Tensor], n_cols: int,
                 deg: Optional[torch.Tensor] = None):
        self.row_ptr = _vec(row_ptr, torch.int64, "row_ptr")
        self.col = _vec(col, torch.int32, "col")
        self.val = None if val is None else _vec(val, torch.float32, "val")
        self.n_rows = row_ptr.numel() - 1
        self.n_cols = int(n_cols)
        self.nnz = col.numel()
        self.deg = deg

    def view(self) -> gsp_csr:
        return gsp_csr(self.n_rows, self.n_cols, self.nnz, self.row_ptr.data_ptr(),
                       self.col.data_ptr() if self.nnz else None,
                       self.val.data_ptr() if (self.val is not None and self.nnz) else None)

    def with_val(self, val: Optional[torch.Tensor]) -> "CSR":
        return CSR(self.row_ptr, self.col, val, self.n_cols, self.deg)


# ---------------------------------------------------------------------------
# a1 / a2
# ---------------------------------------------------------------------------

def gsp_coo_to_csr(n: int, src: torch.Tensor, dst: torch.Tensor, w: Optional[torch.Tensor] = None,
                   undirected: bool = True, fill: float = 1.0, stream=None) -> CSR:
    """COO edge list (device int32/int64) -> canonical CSR of A + fill*I (gsp.h a1)."""
    if src.dtype != dst.dtype or src.dtype not in (torch.int32, torch.int64):
        raise TypeError("src/dst must both be int32 or int64")
    _vec(src, src.dtype, "src")
    _vec(dst, dst.dtype, "dst")
    if w is not None:
        _vec(w, torch.float32, "w")
    m = src.numel()
    if dst.numel() != m or (w is not None and w.numel() != m):
        raise ValueError("src, dst (and w) must have the same length")
    flags = GSP_UNDIRECTED if undirected else 0
    wsb = ctypes.c_size_t(0)
    nmax = ctypes.c_int64(0)
    _check(lib().gsp_coo_to_csr_workspace(n, m, flags, fill, ctypes.byref(wsb), ctypes.byref(nmax)),
           "gsp_coo_to_csr_workspace")
    dev = src.device
    ws = torch.empty(wsb.value + 256, dtype=torch.uint8, device=dev)
    wsp = (ws.data_ptr() + 255) // 256 * 256
    row_ptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    col = torch.empty(max(nmax.value, 1), dtype=torch.int32, device=dev)
    val = torch.empty(max(nmax.value, 1), dtype=torch.float32, device=dev)
    nnz = ctypes.c_int64(0)
    _check(lib().gsp_coo_to_csr(n, m, _ptr(src), _ptr(dst), GSP_I64 if src.dtype == torch.int64 else GSP_I32,
                                _ptr(w), flags, fill, _ptr(row_ptr), _ptr(col), _ptr(val), ctypes.byref(nnz),
                                ctypes.c_void_p(wsp), wsb.value, _stream(stream)), "gsp_coo_to_csr")
    k = nnz.value
    del ws
    return CSR(row_ptr, col[:k], val[:k], n)


def gsp_sym_normalize(a: CSR, in_place: bool = False, keep_deg: bool = True, stream=None) -> CSR:
    """A^ = D~^-1/2 A~ D~^-1/2 (gsp.h a2).  Returns a CSR sharing the structure,
    with the normalised values and (keep_deg) the fp64 degrees in .deg; with
    keep_deg=False the degrees live in a workspace only (deg_out = NULL)."""
    if a.val is None:
        raise ValueError("gsp_sym_normalize needs A~ values")
    out = a.val if in_place else torch.empty_like(a.val)
    v = a.view()
    if keep_deg:
        deg = torch.empty(max(a.n_rows, 1), dtype=torch.float64, device=a.row_ptr.device)
        _check(lib().gsp_sym_normalize(ctypes.byref(v), _ptr(out), _ptr(deg), None, 0, _stream(stream)),
               "gsp_sym_normalize")
        return CSR(a.row_ptr, a.col, out, a.n_cols, deg[:a.n_rows])
    nb = ctypes.c_size_t(0)
    _check(lib().gsp_sym_normalize_workspace(ctypes.byref(v), ctypes.byref(nb)), "gsp_sym_normalize_workspace")
    ws = torch.empty(max(nb.value // 8, 1), dtype=torch.float64, device=a.row_ptr.device)
    _check(lib().gsp_sym_normalize(ctypes.byref(v), _ptr(out), None, _ptr(ws), nb.value, _stream(stream)),
           "gsp_sym_normalize")
    return CSR(a.row_ptr, a.col, out, a.n_cols, None)


def gsp_set_flags(flags: int) -> None:
    """Thread-local library flags (gsp.h): GSP_VALIDATE checks logits / el / er
    for NaN / Inf before compute (GSP_ERR_NONFINITE)."""
    _check(lib().gsp_set_flags(int(flags)), "gsp_set_flags")


def gsp_get_flags() -> int:
    return int(lib().gsp_get_flags())


# ---------------------------------------------------------------------------
# a3
# ---------------------------------------------------------------------------

def gsp_spmm(a: CSR, x: torch.Tensor, f: Optional[int] = None, y: Optional[torch.Tensor] = None, stream=None,
             slab_cols: int = 0, block_nnz: int = 0) -> torch.Tensor:
    """Y = A X (gsp.h a3).  x: [n_cols, >= f] fp32 (row stride = ld)."""
    x, ldx = _mat(x, "x")
    f = x.shape[1] if f is None else int(f)
    if y is None:
        y = empty_features(a.n_rows, f, x.device)
    y, ldy = _mat(y, "y")
    _rows(x, a.n_cols, "x"), _rows(y, a.n_rows, "y"), _width(x, f, "x"), _width(y, f, "y")
    v = a.view()
    if slab_cols or block_nnz:
        o = gsp_spmm_opts(slab_cols, block_nnz)
        st = lib().gsp_spmm_ex(ctypes.byref(v), _ptr(x), f, ldx, _ptr(y), ldy, ctypes.byref(o), _stream(stream))
        _check(st, "gsp_spmm_ex")
    else:
        _check(lib().gsp_spmm(ctypes.byref(v), _ptr(x), f, ldx, _ptr(y), ldy, _stream(stream)), "gsp_spmm")
    return y


gsp_spmm_ex = gsp_spmm

REDUCE = {"sum": 0, "mean": 1, "max": 2, "min": 3}


def gsp_spmm_f16(a: CSR, x: torch.Tensor, f: Optional[int] = None, y: Optional[torch.Tensor] = None,
                 stream=None) -> torch.Tensor:
    """y (fp32) = A x with x stored in fp16 (gsp.h gsp_spmm_f16; fp32 arithmetic)."""
    if x.dtype != torch.float16 or x.dim() != 2 or x.stride(1) != 1:
        raise TypeError("x must be a 2-D float16 tensor with unit column stride")
    f = x.shape[1] if f is None else f
    if y is None:
        y = empty_features(a.n_rows, f, x.device)
    y, ldy = _mat(y, "y")
    _rows(x, a.n_cols, "x"), _rows(y, a.n_rows, "y"), _width(x, f, "x"), _width(y, f, "y")
    v = a.view()
    _check(lib().gsp_spmm_f16(ctypes.byref(v), _ptr(x), f, x.stride(0), _ptr(y), ldy, _stream(stream)), "gsp_spmm_f16")
    return y


def gsp_gspmm(a: CSR, x: torch.Tensor, reduce: str = "sum", f: Optional[int] = None,
              y: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """GSpMM with reduce in {sum, mean, max, min}; psi = mul by a.val (copy if None)."""
    x, ldx = _mat(x, "x")
    f = x.shape[1] if f is None else int(f)
    if y is None:
        y = empty_features(a.n_rows, f, x.device)
    y, ldy = _mat(y, "y")
    _rows(x, a.n_cols, "x"), _rows(y, a.n_rows, "y"), _width(x, f, "x"), _width(y, f, "y")
    v = a.view()
    _check(lib().gsp_gspmm(ctypes.byref(v), REDUCE[reduce], _ptr(x), f, ldx, _ptr(y), ldy, _stream(stream)),
           "gsp_gspmm")
    return y


def gsp_spmm_plan_info(a: CSR, x: torch.Tensor, f: Optional[int] = None, slab_cols: int = 0, block_nnz: int = 0):
    """(launches, slab_cols, tail_slab_cols) gsp_spmm would use (host only)."""
    x, ldx = _mat(x, "x")
    f = x.shape[1] if f is None else int(f)
    o = gsp_spmm_opts(slab_cols, block_nnz)
    n, sc, tc = ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_int32(0)
    v = a.view()
    _check(lib().gsp_spmm_plan_info(ctypes.byref(v), _ptr(x), f, ldx, ctypes.byref(o), ctypes.byref(n),
                                    ctypes.byref(sc), ctypes.byref(tc)), "gsp_spmm_plan_info")
    return n.value, sc.value, tc.value


# ---------------------------------------------------------------------------
# a4 - a7
# ---------------------------------------------------------------------------

def gsp_edge_softmax(a: CSR, logits: torch.Tensor, heads: int, alpha: Optional[torch.Tensor] = None,
                     stream=None) -> torch.Tensor:
    """Row-wise edge softmax per head (gsp.h a6); logits [nnz, heads] (alpha may be logits)."""
    _vec(logits, torch.float32, "logits")
    if alpha is None:
        alpha = torch.empty_like(logits)
    _vec(alpha, torch.float32, "alpha")
    _numel(logits, a.nnz * heads, "logits"), _numel(alpha, a.nnz * heads, "alpha")
    v = a.view()
    _check(lib().gsp_edge_softmax(ctypes.byref(v), heads, _ptr(logits), _ptr(alpha), _stream(stream)),
           "gsp_edge_softmax")
    return alpha


def gsp_multihead_spmm(a: CSR, alpha: torch.Tensor, z: torch.Tensor, heads: int, d: int,
                       y: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Y[u,h,:] = sum_e alpha[e,h] Z[v,h,:] (gsp.h a7).  z: [n_cols, >= heads*d]."""
    _vec(alpha, torch.float32, "alpha")
    z, ldz = _mat(z, "z")
    if y is None:
        y = empty_features(a.n_rows, heads * d, z.device)
    y, ldy = _mat(y, "y")
    _numel(alpha, a.nnz * heads, "alpha"), _rows(z, a.n_cols, "z"), _rows(y, a.n_rows, "y")
    _width(z, heads * d, "z"), _width(y, heads * d, "y")
    v = a.view()
    _check(lib().gsp_multihead_spmm(ctypes.byref(v), heads, _ptr(alpha), _ptr(z), d, ldz, _ptr(y), ldy,
                                    _stream(stream)), "gsp_multihead_spmm")
    return y


def gsp_attn_project(z: torch.Tensor, a_l: torch.Tensor, a_r: torch.Tensor, heads: int, d: int,
                     el: Optional[torch.Tensor] = None, er: Optional[torch.Tensor] = None, stream=None):
    """(el, er) [n, heads] with el[u,h] = a_l[h] . z[u,h,:] (gsp.h a4)."""
    z, ldz = _mat(z, "z")
    n = z.shape[0]
    _vec(a_l, torch.float32, "a_l")
    _vec(a_r, torch.float32, "a_r")
    el = torch.empty((n, heads), dtype=torch.float32, device=z.device) if el is None else el
    er = torch.empty((n, heads), dtype=torch.float32, device=z.device) if er is None else er
    _width(z, heads * d, "z"), _numel(a_l, heads * d, "a_l"), _numel(a_r, heads * d, "a_r")
    _numel(el, n * heads, "el"), _numel(er, n * heads, "er")
    _check(lib().gsp_attn_project(n, heads, d, _ptr(z), ldz, _ptr(a_l), _ptr(a_r), _ptr(el), _ptr(er),
                                  _stream(stream)), "gsp_attn_project")
    return el, er


def gsp_gat_workspace(a: CSR, heads: int) -> int:
    n = ctypes.c_size_t(0)
    v = a.view()
    _check(lib().gsp_gat_workspace(ctypes.byref(v), heads, ctypes.byref(n)), "gsp_gat_workspace")
    return n.value


def _gat_ws(a: CSR, heads: int, device, ws: Optional[torch.Tensor]) -> torch.Tensor:
    need = gsp_gat_workspace(a, heads)
    if ws is None or ws.numel() < need:
        ws = torch.empty(max(need, 16), dtype=torch.uint8, device=device)
    return ws


def gsp_gat_aggregate(a: CSR, el: torch.Tensor, er: torch.Tensor, z: torch.Tensor, heads: int, d: int,
                      negative_slope: float = 0.2, y: Optional[torch.Tensor] = None, alpha_out=None,
                      ws: Optional[torch.Tensor] = None, single_launch: bool = False, stream=None):
    """Fused LeakyReLU score -> edge softmax -> multi-head SpMM (gsp.h a5+a6+a7).
    alpha_out: None, True (allocate) or a [nnz, heads] tensor.  Returns y or (y, alpha).
    ws: statistics workspace (allocated when None); single_launch=True passes no
    workspace, so the statistics are reduced inside the aggregate kernel."""
    _vec(el, torch.float32, "el")
    _vec(er, torch.float32, "er")
    z, ldz = _mat(z, "z")
    if y is None:
        y = empty_features(a.n_rows, heads * d, z.device)
    y, ldy = _mat(y, "y")
    want = alpha_out is not None
    if alpha_out is True:
        alpha_out = torch.empty((a.nnz, heads), dtype=torch.float32, device=z.device)
    _numel(el, a.n_rows * heads, "el"), _numel(er, a.n_cols * heads, "er"), _rows(z, a.n_cols, "z")
    _rows(y, a.n_rows, "y"), _width(z, heads * d, "z"), _width(y, heads * d, "y")
    if want:
        _numel(alpha_out, a.nnz * heads, "alpha_out")
    ws = None if single_launch else _gat_ws(a, heads, z.device, ws)
    v = a.view()
    _check(lib().gsp_gat_aggregate(ctypes.byref(v), heads, _ptr(el), _ptr(er), float(negative_slope), _ptr(z), d,
                                   ldz, _ptr(y), ldy, _ptr(alpha_out if want else None), _ptr(ws),
                                   0 if ws is None else ws.numel(), _stream(stream)), "gsp_gat_aggregate")
    return (y, alpha_out) if want else y


# ---------------------------------------------------------------------------
# multi-GPU partition
# ---------------------------------------------------------------------------

def gsp_partition_rows(a: CSR, parts: int, stream=None):
    """(host list of parts+1 row bounds, device int64 tensor of the same)."""
    dev = torch.empty(parts + 1, dtype=torch.int64, device=a.row_ptr.device)
    host = (ctypes.c_int64 * (parts + 1))()
    v = a.view()
    _check(lib().gsp_partition_rows(ctypes.byref(v), parts, _ptr(dev), host, _stream(stream)),
           "gsp_partition_rows")
    return list(host), dev


def gsp_csr_slice(a: CSR, bounds, rank: int, rows_padded: int, stream=None) -> CSR:
    """Rows of `rank` with columns remapped into the padded all-gather layout."""
    parts = len(bounds) - 1
    hb = (ctypes.c_int64 * (parts + 1))(*[int(b) for b in bounds])
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    rp_host = a.row_ptr[[r0, r1]].tolist()
    k = rp_host[1] - rp_host[0]
    dev = a.row_ptr.device
    rp = torch.empty(r1 - r0 + 1, dtype=torch.int64, device=dev)
    col = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
    val = torch.empty(max(k, 1), dtype=torch.float32, device=dev) if a.val is not None else None
    v = a.view()
    _check(lib().gsp_csr_slice(ctypes.byref(v), hb, parts, rank, rows_padded, _ptr(rp), _ptr(col), _ptr(val),
                               _stream(stream)), "gsp_csr_slice")
    return CSR(rp, col[:k], None if val is None else val[:k], parts * rows_padded)


class ColBlocks:
    """Column blocks of a CSR (gsp_csr_colblock): the device workspace that
    holds them and the borrowed gsp_csr views of the blocks."""

    def __init__(self, a: CSR, bounds, ws: torch.Tensor, views):
        self.a, self.bounds, self.ws, self.views = a, list(bounds), ws, views
        self.n_rows, self.n_cols = a.n_rows, a.n_cols
        self.nnz = [v.nnz for v in views]

    def __len__(self):
        return len(self.views)

    def block(self, k: int) -> CSR:
        """Block k as a CSR of torch views into the workspace."""
        v, base = self.views[k], self.ws.data_ptr()

        def sub(ptr, count, dtype, esize):
            off = ptr - base
            return self.ws[off:off + count * esize].view(dtype)
        rp = sub(v.row_ptr, v.n_rows + 1, torch.int64, 8)
        if v.nnz == 0:
            col = torch.empty(0, dtype=torch.int32, device=rp.device)
            val = None if self.a.val is None else torch.empty(0, dtype=torch.float32, device=rp.device)
        else:
            col = sub(v.col_idx, v.nnz, torch.int32, 4)
            val = sub(v.val, v.nnz, torch.float32, 4) if v.val else None
        return CSR(rp, col, val, v.n_cols)


L2_BYTES = 126 << 20  # B200 L2


def colblock_bounds(a: CSR, f: int, slab_cols: int = 128):
    """Column bounds for gsp_spmm_blocked: two blocks when one slab of X
    (n_cols x slab_cols fp32) overflows ~2/3 of the L2 but two halves fit it,
    and rows are long enough (>= 32 entries on average) that halving them
    does not cost more per-row work than the better L2 hit rate saves
    (measured: C4 4.44 -> 3.9-4.0 ms; C5, whose slab is 3x the
    L2 with 20-entry rows, is slower blocked); else one block."""
    slab = a.n_cols * min(slab_cols, max(int(f), 1)) * 4
    if 2 * L2_BYTES // 3 < slab <= 2 * L2_BYTES and a.nnz >= 32 * max(a.n_rows, 1):
        return [0, a.n_cols // 2, a.n_cols]
    return [0, a.n_cols]


def gsp_csr_colblock(a: CSR, bounds, stream=None) -> ColBlocks:
    """A = sum_k A_k, A_k = the entries with column in [bounds[k], bounds[k+1])
    (gsp.h column blocks); a one-off per graph (one stream sync)."""
    k = len(bounds) - 1
    v = a.view()
    nb = ctypes.c_size_t(0)
    _check(lib().gsp_csr_colblock_workspace(ctypes.byref(v), k, ctypes.byref(nb)), "gsp_csr_colblock_workspace")
    ws = torch.empty(nb.value, dtype=torch.uint8, device=a.row_ptr.device)
    hb = (ctypes.c_int64 * (k + 1))(*[int(b) for b in bounds])
    out = (gsp_csr * k)()
    _check(lib().gsp_csr_colblock(ctypes.byref(v), hb, k, _ptr(ws), nb.value, out, _stream(stream)),
           "gsp_csr_colblock")
    return ColBlocks(a, bounds, ws, [out[i] for i in range(k)])


def gsp_spmm_blocked(blocks: ColBlocks, x: torch.Tensor, f: Optional[int] = None, y: Optional[torch.Tensor] = None,
                     stream=None) -> torch.Tensor:
    """Y = sum_k A_k X over column blocks (gsp.h gsp_spmm_blocked)."""
    x, ldx = _mat(x, "x")
    f = x.shape[1] if f is None else int(f)
    if y is None:
        y = empty_features(blocks.n_rows, f, x.device)
    y, ldy = _mat(y, "y")
    _rows(x, blocks.n_cols, "x"), _rows(y, blocks.n_rows, "y"), _width(x, f, "x"), _width(y, f, "y")
    arr = (gsp_csr * len(blocks.views))(*blocks.views)
    _check(lib().gsp_spmm_blocked(arr, len(blocks.views), _ptr(x), f, ldx, _ptr(y), ldy, _stream(stream)),
           "gsp_spmm_blocked")
    return y


def gsp_spmm_accumulate(a: CSR, x: torch.Tensor, acc: torch.Tensor, coef: float, f: Optional[int] = None,
                        t: Optional[torch.Tensor] = None, src: Optional[torch.Tensor] = None, src_coef: float = 0.0,
                        stream=None):
    """One propagation step: t = A x (if t given); acc = coef*t + (src_coef*src if src else acc)."""
    x, ldx = _mat(x, "x")
    f = x.shape[1] if f is None else int(f)
    acc, ldacc = _mat(acc, "acc")
    ldt = _mat(t, "t")[1] if t is not None else 0
    ldsrc = _mat(src, "src")[1] if src is not None else 0
    v = a.view()
    _check(lib().gsp_spmm_accumulate(ctypes.byref(v), _ptr(x), f, ldx, _ptr(t), ldt, _ptr(acc), ldacc, coef,
                                     _ptr(src), ldsrc, src_coef, _stream(stream)), "gsp_spmm_accumulate")
    return acc


def gsp_propagate(a: CSR, x: torch.Tensor, theta, f: Optional[int] = None, y: Optional[torch.Tensor] = None,
                  ws: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """y = sum_k theta_k A^k x (K = len(theta) - 1 >= 1)."""
    x, ldx = _mat(x, "x")
    f = x.shape[1] if f is None else int(f)
    th = (ctypes.c_double * len(theta))(*[float(t) for t in theta])
    if y is None:
        y = empty_features(a.n_rows, f, x.device)
    y, ldy = _mat(y, "y")
    n = ctypes.c_size_t(0)
    v = a.view()
    _check(lib().gsp_propagate_workspace(ctypes.byref(v), f, len(theta) - 1, ctypes.byref(n)),
           "gsp_propagate_workspace")
    if n.value and (ws is None or ws.numel() < n.value):
        ws = torch.empty(n.value, dtype=torch.uint8, device=x.device)
    _check(lib().gsp_propagate(ctypes.byref(v), _ptr(x), f, ldx, len(theta) - 1, th, _ptr(y), ldy,
                               _ptr(ws) if n.value else None, n.value, _stream(stream)), "gsp_propagate")
    return y


# ---------------------------------------------------------------------------
# NEXT-3: GAT backward
# ---------------------------------------------------------------------------

def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1) + 256, dtype=torch.uint8, device=device)


def _aligned(t: torch.Tensor):
    return ctypes.c_void_p((t.data_ptr() + 255) // 256 * 256)


def gsp_csr_transpose(a: CSR, stream=None):
    """(A^T as CSR, perm int32 [nnz]): entry e' of A^T is entry perm[e'] of A."""
    n = ctypes.c_size_t(0)
    v = a.view()
    _check(lib().gsp_csr_transpose_workspace(ctypes.byref(v), ctypes.byref(n)), "gsp_csr_transpose_workspace")
    dev = a.row_ptr.device
    ws = _ws(n.value, dev)
    rp = torch.empty(a.n_cols + 1, dtype=torch.int64, device=dev)
    ct = torch.empty(max(a.nnz, 1), dtype=torch.int32, device=dev)
    pm = torch.empty(max(a.nnz, 1), dtype=torch.int32, device=dev)
    _check(lib().gsp_csr_transpose(ctypes.byref(v), _ptr(rp), _ptr(ct), _ptr(pm), _aligned(ws), n.value,
                                   _stream(stream)), "gsp_csr_transpose")
    return CSR(rp, ct[:a.nnz], None, a.n_rows), pm[:a.nnz]


def gsp_sddmm(a: CSR, p: torch.Tensor, q: torch.Tensor, heads: int = 1, d: Optional[int] = None,
              out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """out [nnz, heads]: out[e,h] = <p[u,h,:], q[v,h,:]>."""
    p, ldp = _mat(p, "p")
    q, ldq = _mat(q, "q")
    d = p.shape[1] // heads if d is None else d
    out = torch.empty((a.nnz, heads), dtype=torch.float32, device=p.device) if out is None else out
    v = a.view()
    _check(lib().gsp_sddmm(ctypes.byref(v), heads, _ptr(p), d, ldp, _ptr(q), ldq, _ptr(out), _stream(stream)),
           "gsp_sddmm")
    return out


def gsp_edge_softmax_backward(a: CSR, alpha: torch.Tensor, dalpha: torch.Tensor, heads: int,
                              ds: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    ds = torch.empty_like(dalpha) if ds is None else ds
    v = a.view()
    _check(lib().gsp_edge_softmax_backward(ctypes.byref(v), heads, _ptr(alpha), _ptr(dalpha), _ptr(ds),
                                           _stream(stream)), "gsp_edge_softmax_backward")
    return ds


def gsp_gat_aggregate_backward(a: CSR, at: CSR, perm: torch.Tensor, el: torch.Tensor, er: torch.Tensor,
                               z: torch.Tensor, dy: torch.Tensor, heads: int, d: int, negative_slope: float = 0.2,
                               stream=None):
    """(dz, d_el, d_er) of gsp_gat_aggregate's output gradient dy."""
    z, ldz = _mat(z, "z")
    dy, lddy = _mat(dy, "dy")
    dz = empty_features(a.n_cols, heads * d, z.device)
    d_el = torch.empty((a.n_rows, heads), dtype=torch.float32, device=z.device)
    d_er = torch.empty((a.n_cols, heads), dtype=torch.float32, device=z.device)
    n = ctypes.c_size_t(0)
    v, vt = a.view(), at.view()
    _check(lib().gsp_gat_backward_workspace(ctypes.byref(v), heads, ctypes.byref(n)), "gsp_gat_backward_workspace")
    ws = _ws(n.value, z.device)
    _check(lib().gsp_gat_aggregate_backward(ctypes.byref(v), ctypes.byref(vt), _ptr(perm), heads, _ptr(el),
                                            _ptr(er), float(negative_slope), _ptr(z), d, ldz, _ptr(dy), lddy,
                                            _ptr(dz), dz.stride(0), _ptr(d_el), _ptr(d_er), _aligned(ws), n.value,
                                            _stream(stream)), "gsp_gat_aggregate_backward")
    return dz, d_el, d_er


def gsp_attn_project_backward(z: torch.Tensor, a_l: torch.Tensor, a_r: torch.Tensor, d_el: torch.Tensor,
                              d_er: torch.Tensor, dz: torch.Tensor, heads: int, d: int, stream=None):
    """dz += d_el a_l + d_er a_r (in place); returns (d_al, d_ar) [heads*d]."""
    z, ldz = _mat(z, "z")
    dz, lddz = _mat(dz, "dz")
    n = z.shape[0]
    d_al = torch.empty(heads * d, dtype=torch.float32, device=z.device)
    d_ar = torch.empty(heads * d, dtype=torch.float32, device=z.device)
    nb = ctypes.c_size_t(0)
    _check(lib().gsp_attn_project_backward_workspace(n, heads, d, ctypes.byref(nb)),
           "gsp_attn_project_backward_workspace")
    ws = _ws(nb.value, z.device)
    _check(lib().gsp_attn_project_backward(n, heads, d, _ptr(z), ldz, _ptr(a_l), _ptr(a_r), _ptr(d_el), _ptr(d_er),
                                           _ptr(dz), lddz, _ptr(d_al), _ptr(d_ar), _aligned(ws), nb.value,
                                           _stream(stream)), "gsp_attn_project_backward")
    return d_al, d_ar


# ---------------------------------------------------------------------------
# NEXT-1: inference layers
# ---------------------------------------------------------------------------

ACT = {"none": 0, "relu": 1, "elu": 2}


def gsp_linear(x: torch.Tensor, w: torch.Tensor, y: Optional[torch.Tensor] = None, ws: Optional[torch.Tensor] = None,
               tensor_cores: bool = True, stream=None) -> torch.Tensor:
    """y = x w (row-major): tcgen05 3xTF32 GEMM when a workspace is passed
    (allocated here unless tensor_cores=False), else fp32 cuBLAS."""
    x, ldx = _mat(x, "x")
    w, ldw = _mat(w, "w")
    n, f_in = x.shape
    f_out = w.shape[1]
    y = empty_features(n, f_out, x.device) if y is None else y
    y, ldy = _mat(y, "y")
    if tensor_cores:
        nb = ctypes.c_size_t(0)
        _check(lib().gsp_linear_workspace(f_in, f_out, ctypes.byref(nb)), "gsp_linear_workspace")
        if ws is None or ws.numel() < nb.value:
            ws = torch.empty(nb.value, dtype=torch.uint8, device=x.device)
    else:
        ws = None
    _check(lib().gsp_linear(n, f_in, _ptr(x), ldx, _ptr(w), ldw, f_out, _ptr(y), ldy, _ptr(ws),
                            0 if ws is None else ws.numel(), _stream(stream)), "gsp_linear")
    return y


def gsp_spmm_bias_act(a: CSR, x: torch.Tensor, bias: Optional[torch.Tensor] = None, act: str = "none",
                      f: Optional[int] = None, y: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    x, ldx = _mat(x, "x")
    f = x.shape[1] if f is None else int(f)
    y = empty_features(a.n_rows, f, x.device) if y is None else y
    y, ldy = _mat(y, "y")
    v = a.view()
    _check(lib().gsp_spmm_bias_act(ctypes.byref(v), _ptr(x), f, ldx, _ptr(bias), ACT[act], _ptr(y), ldy,
                                   _stream(stream)), "gsp_spmm_bias_act")
    return y


def gsp_gcn_layer(a: CSR, x: torch.Tensor, w: torch.Tensor, bias: Optional[torch.Tensor] = None, act: str = "relu",
                  y: Optional[torch.Tensor] = None, ws: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """y = act(A (x w) + bias)  (Eq. gcn_layer)."""
    x, ldx = _mat(x, "x")
    f_in, f_out = w.shape
    y = empty_features(a.n_rows, f_out, x.device) if y is None else y
    y, ldy = _mat(y, "y")
    nb = ctypes.c_size_t(0)
    _check(lib().gsp_gcn_layer_workspace(a.n_cols, f_in, f_out, ctypes.byref(nb)), "gsp_gcn_layer_workspace")
    if ws is None or ws.numel() < nb.value:
        ws = torch.empty(nb.value, dtype=torch.uint8, device=x.device)
    v = a.view()
    _check(lib().gsp_gcn_layer(ctypes.byref(v), _ptr(x), f_in, ldx, _ptr(w.contiguous()), f_out, _ptr(bias),
                               ACT[act], _ptr(y), ldy, _ptr(ws), ws.numel(), _stream(stream)), "gsp_gcn_layer")
    return y


def gsp_gat_aggregate_bias_act(a: CSR, el: torch.Tensor, er: torch.Tensor, z: torch.Tensor, heads: int, d: int,
                               bias: Optional[torch.Tensor] = None, act: str = "none", negative_slope: float = 0.2,
                               y: Optional[torch.Tensor] = None, ws: Optional[torch.Tensor] = None,
                               single_launch: bool = False, stream=None) -> torch.Tensor:
    """gsp_gat_aggregate with act(Y + bias) fused; ws / single_launch as there."""
    z, ldz = _mat(z, "z")
    y = empty_features(a.n_rows, heads * d, z.device) if y is None else y
    y, ldy = _mat(y, "y")
    _numel(el, a.n_rows * heads, "el"), _numel(er, a.n_cols * heads, "er"), _rows(z, a.n_cols, "z")
    _rows(y, a.n_rows, "y"), _width(z, heads * d, "z"), _width(y, heads * d, "y")
    if bias is not None:
        _numel(bias, heads * d, "bias")
    ws = None if single_launch else _gat_ws(a, heads, z.device, ws)
    v = a.view()
    _check(lib().gsp_gat_aggregate_bias_act(ctypes.byref(v), heads, _ptr(el), _ptr(er), float(negative_slope),
                                            _ptr(z), d, ldz, _ptr(bias), ACT[act], _ptr(y), ldy, _ptr(ws),
                                            0 if ws is None else ws.numel(), _stream(stream)),
           "gsp_gat_aggregate_bias_act")
    return y


def version() -> int:
    return lib().gsp_version()
