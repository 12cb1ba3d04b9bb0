"""fp64 CPU oracle for the CogDL (arXiv 2103.00959) sparse-operator hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  It shares no
code with the CUDA path (paper_2103_00959_b200/) and the product never imports
it.  The arithmetic lives in oracle.c (plain fp64 C loops, each function citing
the PAPER.md passage it follows); this module only marshals numpy arrays.

Parity status: every function is pinned by
tests/test_oracle_pins.py against dense NumPy linear algebra, closed forms,
brute force over all small graphs, the SPEC.md worked examples
(tests/golden/*.json) and invariants.  No function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def _compile(out, extra):
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, *extra, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, out)
    return out


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (IEEE double, no FMA contraction), and the
    same source with -fopenmp as liboracle_omp.so (row loops of spmm /
    multihead_spmm on all host cores; identical per-row arithmetic)."""
    if force:
        for p in (_LIB, _LIB_OMP):
            if os.path.exists(p):
                os.remove(p)
    _compile(_LIB_OMP, ["-fopenmp"])
    return _compile(_LIB, [])


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def usable_cores() -> int:
    return len(os.sched_getaffinity(0))


_lib = None
_lib_omp = None


def lib_omp():
    """The OpenMP build (same oracle.c); threads = OMP_NUM_THREADS or all usable cores."""
    global _lib_omp
    if _lib_omp is None:
        build()
        os.environ.setdefault("OMP_NUM_THREADS", str(usable_cores()))
        L = ctypes.CDLL(_LIB_OMP)
        P, I = ctypes.c_void_p, ctypes.c_int64
        L.orc_spmm.argtypes = [I, I, P, P, P, P, I, I, P, P, I]
        L.orc_multihead_spmm.argtypes = [I, I, P, P, I, P, P, I, I, P, P, I]
        L.orc_spmm.restype = L.orc_multihead_spmm.restype = ctypes.c_int
        _lib_omp = L
    return _lib_omp
_i64p = ctypes.POINTER(ctypes.c_int64)


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        P = ctypes.c_void_p
        I = ctypes.c_int64
        L.orc_build_csr.argtypes = [I, I, P, P, P, ctypes.c_int, ctypes.c_float, P, P, P, I, P]
        L.orc_sym_norm.argtypes = [I, P, P, P, P, P, P]
        L.orc_spmm.argtypes = [I, I, P, P, P, P, I, I, P, P, I]
        L.orc_gspmm.argtypes = [I, I, P, P, P, P, I, I, ctypes.c_int, P, I]
        L.orc_propagate.argtypes = [I, P, P, P, P, I, I, I, P, P, P, I]
        L.orc_ppr_coeffs.argtypes = [ctypes.c_double, I, P]
        L.orc_edge_softmax.argtypes = [I, I, P, I, P, P]
        L.orc_gat_scores.argtypes = [I, I, P, P, I, P, P, ctypes.c_double, P]
        L.orc_multihead_spmm.argtypes = [I, I, P, P, I, P, P, I, I, P, P, I]
        L.orc_attn_project.argtypes = [I, I, I, I, P, I, P, P, P, P, P, P]
        L.orc_partition_rows.argtypes = [I, P, I, P]
        L.orc_sddmm.argtypes = [I, P, P, I, I, P, I, P, I, P]
        L.orc_csr_transpose.argtypes = [I, I, P, P, P, P, P]
        L.orc_edge_softmax_backward.argtypes = [I, P, I, P, P, P]
        L.orc_gat_backward.argtypes = [I, P, P, I, P, P, ctypes.c_double, P, I, I, P, I, P, P, P, P]
        L.orc_attn_project_backward.argtypes = [I, I, I, P, I, P, P, P, P, P, P, P]
        L.orc_linear.argtypes = [I, I, P, I, I, P, I, P, P, P, I]
        L.orc_gcn_layer.argtypes = [I, I, P, P, P, P, I, I, P, I, P, ctypes.c_int, P, P, I]
        L.orc_bias_act.argtypes = [I, I, P, I, P, ctypes.c_int]
        L.orc_csr_slice.argtypes = [I, P, P, P, P, I, I, I, P, P, P]
        for f in ("orc_build_csr", "orc_sym_norm", "orc_spmm", "orc_gspmm", "orc_propagate", "orc_ppr_coeffs", "orc_edge_softmax", "orc_gat_scores",
                  "orc_multihead_spmm", "orc_attn_project", "orc_partition_rows", "orc_csr_slice", "orc_sddmm",
                  "orc_csr_transpose", "orc_edge_softmax_backward", "orc_gat_backward", "orc_attn_project_backward",
                  "orc_linear", "orc_gcn_layer", "orc_bias_act"):
            getattr(L, f).restype = ctypes.c_int
    return _lib


class OracleError(RuntimeError):
    CODES = {-1: "invalid argument", -2: "index out of range", -3: "negative weight",
             -4: "non-finite weight", -5: "capacity", -6: "out of memory"}

    def __init__(self, code):
        super().__init__(f"oracle error {code}: {self.CODES.get(code, '?')}")
        self.code = code


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _chk(rc):
    if rc != 0:
        raise OracleError(rc)


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


class CSR:
    """Host CSR (row_ptr int64[n+1], col int32[nnz], val float32[nnz])."""

    def __init__(self, n, row_ptr, col, val):
        self.n, self.row_ptr, self.col, self.val = n, row_ptr, col, val

    @property
    def nnz(self):
        return int(self.row_ptr[-1])

    def dense(self, vals=None):
        v = self.val if vals is None else vals
        A = np.zeros((self.n, self.n), dtype=np.float64)
        for u in range(self.n):
            for e in range(self.row_ptr[u], self.row_ptr[u + 1]):
                A[u, self.col[e]] += v[e]
        return A


def build_csr(n, src, dst, w=None, undirected=True, fill=1.0) -> CSR:
    """Canonical CSR of A~ = A + fill*I (oracle.c §1)."""
    src = _c(src, np.int64)
    dst = _c(dst, np.int64)
    w = _c(w, np.float32)
    m = src.size
    cap = m * (2 if undirected else 1) + (n if fill != 0 else 0)
    row_ptr = np.zeros(n + 1, np.int64)
    col = np.zeros(max(cap, 1), np.int32)
    val = np.zeros(max(cap, 1), np.float32)
    nnz = ctypes.c_int64(0)
    _chk(lib().orc_build_csr(n, m, _p(src), _p(dst), _p(w), int(bool(undirected)), float(fill),
                             _p(row_ptr), _p(col), _p(val), cap, ctypes.byref(nnz)))
    k = nnz.value
    return CSR(n, row_ptr, col[:k].copy(), val[:k].copy())


def sym_norm(g: CSR):
    """(deg fp64[n], a64 fp64[nnz], a32 fp32[nnz]) of A^ = D~^-1/2 A~ D~^-1/2 (oracle.c §2)."""
    deg = np.zeros(g.n, np.float64)
    a64 = np.zeros(g.nnz, np.float64)
    a32 = np.zeros(g.nnz, np.float32)
    _chk(lib().orc_sym_norm(g.n, _p(g.row_ptr), _p(g.col), _p(_c(g.val, np.float32)), _p(deg), _p(a64), _p(a32)))
    return deg, a64, a32


def spmm(row_ptr, col, a, x, f=None, r0=0, r1=None, want_cond=True, omp=False):
    """(y, cond) fp64 [r1-r0, f] for Y = A X over rows [r0, r1) (oracle.c §3);
    omp=True runs the same rows on all host cores (liboracle_omp.so)."""
    row_ptr = _c(row_ptr, np.int64)
    col = _c(col, np.int32)
    a = _c(a, np.float64)
    x = np.ascontiguousarray(x, dtype=np.float32)
    n = row_ptr.size - 1
    r1 = n if r1 is None else r1
    f = x.shape[1] if f is None else f
    y = np.zeros((r1 - r0, max(f, 1)), np.float64)
    cond = np.zeros_like(y) if want_cond else None
    _chk((lib_omp() if omp else lib()).orc_spmm(r0, r1, _p(row_ptr), _p(col), _p(a), _p(x), f, x.shape[1], _p(y), _p(cond), y.shape[1]))
    return y[:, :f], (cond[:, :f] if want_cond else None)


REDUCE = {"sum": 0, "mean": 1, "max": 2, "min": 3}


def gspmm(row_ptr, col, a, x, reduce="sum", f=None, r0=0, r1=None):
    """y fp64 [r1-r0, f] = phi_e psi(a_e, x[col_e]) (oracle.c §3b); a None -> copy."""
    row_ptr = _c(row_ptr, np.int64)
    col = _c(col, np.int32)
    a = _c(a, np.float64)
    x = np.ascontiguousarray(x, dtype=np.float32)
    n = row_ptr.size - 1
    r1 = n if r1 is None else r1
    f = x.shape[1] if f is None else f
    y = np.zeros((r1 - r0, max(f, 1)), np.float64)
    _chk(lib().orc_gspmm(r0, r1, _p(row_ptr), _p(col), _p(a), _p(x), f, x.shape[1], REDUCE[reduce], _p(y),
                         y.shape[1]))
    return y[:, :f]


def propagate(row_ptr, col, a, x, theta, f=None, want_cond=True):
    """(y, cond) fp64 [n, f] = sum_k theta_k A^k x (oracle.c §3c)."""
    row_ptr = _c(row_ptr, np.int64)
    col = _c(col, np.int32)
    a = _c(a, np.float64)
    x = np.ascontiguousarray(x, dtype=np.float32)
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    n = row_ptr.size - 1
    f = x.shape[1] if f is None else f
    y = np.zeros((n, max(f, 1)), np.float64)
    cond = np.zeros_like(y) if want_cond else None
    _chk(lib().orc_propagate(n, _p(row_ptr), _p(col), _p(a), _p(x), f, x.shape[1], theta.size - 1, _p(theta), _p(y),
                             _p(cond), y.shape[1]))
    return y[:, :f], (cond[:, :f] if want_cond else None)


def ppr_coeffs(alpha, K):
    th = np.zeros(K + 1, np.float64)
    _chk(lib().orc_ppr_coeffs(float(alpha), K, _p(th)))
    return th


def edge_softmax(row_ptr, logits, heads=1, r0=0, r1=None):
    """alpha fp64 [nnz, heads] (oracle.c §4); entries outside [r0, r1) stay 0."""
    row_ptr = _c(row_ptr, np.int64)
    lg = np.ascontiguousarray(logits, dtype=np.float64).reshape(-1)
    n = row_ptr.size - 1
    r1 = n if r1 is None else r1
    alpha = np.zeros(lg.size, np.float64)
    _chk(lib().orc_edge_softmax(r0, r1, _p(row_ptr), heads, _p(lg), _p(alpha)))
    return alpha.reshape(-1, heads)


def gat_scores(row_ptr, col, el, er, heads, slope=0.2, r0=0, r1=None):
    """s fp64 [nnz, heads] = LeakyReLU(el[u] + er[v]) (oracle.c §5)."""
    row_ptr = _c(row_ptr, np.int64)
    col = _c(col, np.int32)
    el = np.ascontiguousarray(el, dtype=np.float32)
    er = np.ascontiguousarray(er, dtype=np.float32)
    n = row_ptr.size - 1
    r1 = n if r1 is None else r1
    s = np.zeros(int(row_ptr[-1]) * heads, np.float64)
    _chk(lib().orc_gat_scores(r0, r1, _p(row_ptr), _p(col), heads, _p(el), _p(er), float(slope), _p(s)))
    return s.reshape(-1, heads)


def multihead_spmm(row_ptr, col, alpha, z, heads, d, r0=0, r1=None, want_cond=True, omp=False):
    """(y, cond) fp64 [r1-r0, heads*d] (oracle.c §6); omp as for spmm."""
    row_ptr = _c(row_ptr, np.int64)
    col = _c(col, np.int32)
    alpha = np.ascontiguousarray(alpha, dtype=np.float64).reshape(-1)
    z = np.ascontiguousarray(z, dtype=np.float32)
    n = row_ptr.size - 1
    r1 = n if r1 is None else r1
    w = heads * d
    y = np.zeros((r1 - r0, max(w, 1)), np.float64)
    cond = np.zeros_like(y) if want_cond else None
    _chk((lib_omp() if omp else lib()).orc_multihead_spmm(r0, r1, _p(row_ptr), _p(col), heads, _p(alpha), _p(z), d, z.shape[1],
                                  _p(y), _p(cond), y.shape[1]))
    return y[:, :w], (cond[:, :w] if want_cond else None)


def attn_project(z, a_l, a_r, heads, d, r0=0, r1=None):
    """(el, er, el_cond, er_cond) fp64 [rows, heads] (oracle.c §7)."""
    z = np.ascontiguousarray(z, dtype=np.float32)
    a_l = np.ascontiguousarray(a_l, dtype=np.float32).reshape(-1)
    a_r = np.ascontiguousarray(a_r, dtype=np.float32).reshape(-1)
    r1 = z.shape[0] if r1 is None else r1
    out = [np.zeros((r1 - r0, heads), np.float64) for _ in range(4)]
    _chk(lib().orc_attn_project(r0, r1, heads, d, _p(z), z.shape[1], _p(a_l), _p(a_r), *[_p(o) for o in out]))
    return tuple(out)


def partition_rows(row_ptr, parts):
    row_ptr = _c(row_ptr, np.int64)
    b = np.zeros(parts + 1, np.int64)
    _chk(lib().orc_partition_rows(row_ptr.size - 1, _p(row_ptr), parts, _p(b)))
    return b


def csr_slice(row_ptr, col, val, bounds, rank, rows_padded):
    row_ptr = _c(row_ptr, np.int64)
    col = _c(col, np.int32)
    val = _c(val, np.float32)
    bounds = _c(bounds, np.int64)
    parts = bounds.size - 1
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    k = int(row_ptr[r1] - row_ptr[r0])
    rp = np.zeros(r1 - r0 + 1, np.int64)
    co = np.zeros(max(k, 1), np.int32)
    vo = np.zeros(max(k, 1), np.float32)
    _chk(lib().orc_csr_slice(row_ptr.size - 1, _p(row_ptr), _p(col), _p(val), _p(bounds), parts, rank,
                             rows_padded, _p(rp), _p(co), _p(vo)))
    return rp, co[:k], vo[:k]


def sddmm(row_ptr, col, p, q, heads=1, d=None):
    """out fp64 [nnz, heads] = per-edge per-head dot(p[u], q[v]) (oracle.c §10a)."""
    row_ptr = _c(row_ptr, np.int64)
    col = _c(col, np.int32)
    p = np.ascontiguousarray(p, dtype=np.float32)
    q = np.ascontiguousarray(q, dtype=np.float32)
    d = p.shape[1] // heads if d is None else d
    out = np.zeros(max(int(row_ptr[-1]) * heads, 1), np.float64)
    _chk(lib().orc_sddmm(row_ptr.size - 1, _p(row_ptr), _p(col), heads, d, _p(p), p.shape[1], _p(q), q.shape[1],
                         _p(out)))
    return out[:int(row_ptr[-1]) * heads].reshape(-1, heads)


def csr_transpose(row_ptr, col, n_cols):
    """(row_ptr_t, col_t, perm) of A^T (oracle.c §10b)."""
    row_ptr = _c(row_ptr, np.int64)
    col = _c(col, np.int32)
    nnz = int(row_ptr[-1])
    rp = np.zeros(n_cols + 1, np.int64)
    ct = np.zeros(max(nnz, 1), np.int32)
    pm = np.zeros(max(nnz, 1), np.int64)
    _chk(lib().orc_csr_transpose(row_ptr.size - 1, n_cols, _p(row_ptr), _p(col), _p(rp), _p(ct), _p(pm)))
    return rp, ct[:nnz], pm[:nnz]


def edge_softmax_backward(row_ptr, alpha, dalpha, heads=1):
    row_ptr = _c(row_ptr, np.int64)
    a = np.ascontiguousarray(alpha, dtype=np.float64).reshape(-1)
    da = np.ascontiguousarray(dalpha, dtype=np.float64).reshape(-1)
    ds = np.zeros(max(a.size, 1), np.float64)
    _chk(lib().orc_edge_softmax_backward(row_ptr.size - 1, _p(row_ptr), heads, _p(a), _p(da), _p(ds)))
    return ds[:a.size].reshape(-1, heads)


def gat_backward(row_ptr, col, el, er, z, dy, heads, d, slope=0.2):
    """(dz [n, H*D], d_el [n, H], d_er [n, H], dt [nnz, H]) fp64 (oracle.c §10d)."""
    row_ptr = _c(row_ptr, np.int64)
    col = _c(col, np.int32)
    el = np.ascontiguousarray(el, dtype=np.float32)
    er = np.ascontiguousarray(er, dtype=np.float32)
    z = np.ascontiguousarray(z, dtype=np.float32)
    dy = np.ascontiguousarray(dy, dtype=np.float32)
    n = row_ptr.size - 1
    dz = np.zeros((n, heads * d), np.float64)
    d_el = np.zeros((n, heads), np.float64)
    d_er = np.zeros((n, heads), np.float64)
    dt = np.zeros(max(int(row_ptr[-1]) * heads, 1), np.float64)
    _chk(lib().orc_gat_backward(n, _p(row_ptr), _p(col), heads, _p(el), _p(er), float(slope), _p(z), d, z.shape[1],
                                _p(dy), dy.shape[1], _p(dz), _p(d_el), _p(d_er), _p(dt)))
    return dz, d_el, d_er, dt[:int(row_ptr[-1]) * heads].reshape(-1, heads)


def attn_project_backward(z, a_l, a_r, d_el, d_er, heads, d):
    """(dz [n, H*D], d_al [H*D], d_ar [H*D]) fp64 (oracle.c §10e)."""
    z = np.ascontiguousarray(z, dtype=np.float32)
    a_l = np.ascontiguousarray(a_l, dtype=np.float32).reshape(-1)
    a_r = np.ascontiguousarray(a_r, dtype=np.float32).reshape(-1)
    d_el = np.ascontiguousarray(d_el, dtype=np.float64)
    d_er = np.ascontiguousarray(d_er, dtype=np.float64)
    n = z.shape[0]
    dz = np.zeros((n, heads * d), np.float64)
    d_al = np.zeros(heads * d, np.float64)
    d_ar = np.zeros(heads * d, np.float64)
    _chk(lib().orc_attn_project_backward(n, heads, d, _p(z), z.shape[1], _p(a_l), _p(a_r), _p(d_el), _p(d_er),
                                         _p(dz), _p(d_al), _p(d_ar)))
    return dz, d_al, d_ar


ACT = {"none": 0, "relu": 1, "elu": 2}


def linear(x, w, bias=None, r0=0, r1=None):
    """(y, cond) fp64 = x W (+ bias) on rows [r0, r1) (oracle.c §11a)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    bias = _c(bias, np.float32)
    r1 = x.shape[0] if r1 is None else r1
    f_in, f_out = w.shape
    y = np.zeros((r1 - r0, max(f_out, 1)), np.float64)
    cond = np.zeros_like(y)
    _chk(lib().orc_linear(r0, r1, _p(x), x.shape[1], f_in, _p(w), f_out, _p(bias), _p(y), _p(cond), y.shape[1]))
    return y[:, :f_out], cond[:, :f_out]


def gcn_layer(row_ptr, col, a, x, w, bias=None, act="relu", r0=0, r1=None):
    """(y, cond) fp64 = act(sum_e a_e x[v] W + b) on rows [r0, r1) (oracle.c §11b)."""
    row_ptr = _c(row_ptr, np.int64)
    col = _c(col, np.int32)
    a = _c(a, np.float64)
    x = np.ascontiguousarray(x, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    bias = _c(bias, np.float32)
    n = row_ptr.size - 1
    r1 = n if r1 is None else r1
    f_in, f_out = w.shape
    y = np.zeros((r1 - r0, max(f_out, 1)), np.float64)
    cond = np.zeros_like(y)
    _chk(lib().orc_gcn_layer(r0, r1, _p(row_ptr), _p(col), _p(a), _p(x), x.shape[1], f_in, _p(w), f_out, _p(bias),
                             ACT[act], _p(y), _p(cond), y.shape[1]))
    return y[:, :f_out], cond[:, :f_out]


def bias_act(y, bias=None, act="none"):
    y = np.array(y, dtype=np.float64, order="C", copy=True)
    bias = _c(bias, np.float32)
    _chk(lib().orc_bias_act(y.shape[0], y.shape[1], _p(y), y.shape[1], _p(bias), ACT[act]))
    return y
