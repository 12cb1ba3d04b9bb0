"""Pins for the fp64 oracle (run with -m "not gpu").

The oracle is checked against things other than itself: dense NumPy/SciPy
linear algebra (a different algorithm and summation order), closed forms,
brute force over every small graph, the SPEC.md worked examples
(tests/golden/spec_examples.json), and invariants that hold at any size.
Each test names the plausible oracle mistake it would catch.
"""
import itertools

import numpy as np
import pytest
import scipy.special

import oracle as orc
from synth import chung_lu, erdos_renyi, features, rmat, uniform, weights


# ---------------------------------------------------------------------------
# helpers: independent dense constructions (NumPy only)
# ---------------------------------------------------------------------------

def dense_adj(n, src, dst, w=None, undirected=True, fill=1.0):
    """A~ = A + fill*I built densely with np.add.at (A2/A4/A5)."""
    A = np.zeros((n, n), np.float64)
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    w = np.ones(src.size) if w is None else np.asarray(w, np.float64)
    np.add.at(A, (src, dst), w)
    if undirected:
        off = src != dst
        np.add.at(A, (dst[off], src[off]), w[off])
    A[np.arange(n), np.arange(n)] += fill
    return A


def dense_norm(A):
    d = A.sum(1)
    with np.errstate(divide="ignore"):
        s = np.where(d > 0, 1.0 / np.sqrt(d), 0.0)
    return s[:, None] * A * s[None, :]


def check_canonical(g):
    assert g.row_ptr[0] == 0 and np.all(np.diff(g.row_ptr) >= 0)
    for u in range(g.n):
        c = g.col[g.row_ptr[u]:g.row_ptr[u + 1]]
        assert np.all(np.diff(c) > 0), "columns not strictly increasing"


# ---------------------------------------------------------------------------
# 1. build (oracle.c §1)
# ---------------------------------------------------------------------------

def test_build_spec_examples(golden):
    for case in golden["spec_examples"]["build"]:
        e = np.array(case["edges"], np.int64).reshape(-1, 2)
        g = orc.build_csr(case["n"], e[:, 0], e[:, 1], case["weights"], case["undirected"], case["fill"])
        assert g.row_ptr.tolist() == case["row_ptr"], case["cite"]
        assert g.col.tolist() == case["col"], case["cite"]
        assert g.val.tolist() == case["val"], case["cite"]


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_build_bruteforce_all_undirected_graphs(n):
    """Every simple undirected graph on n <= 5 nodes (1,024 at n = 5) vs a dense
    construction.  Catches dropped reverse edges, missing loops, bad row_ptr."""
    pairs = list(itertools.combinations(range(n), 2))
    for mask in range(1 << len(pairs)):
        e = np.array([p for i, p in enumerate(pairs) if mask >> i & 1], np.int64).reshape(-1, 2)
        g = orc.build_csr(n, e[:, 0], e[:, 1], None, True, 1.0)
        check_canonical(g)
        np.testing.assert_array_equal(g.dense(), dense_adj(n, e[:, 0], e[:, 1]))
        assert g.nnz == 2 * len(e) + n


def test_build_bruteforce_directed_n3():
    """All 64 directed loop-free graphs on 3 nodes, with and without fill."""
    pairs = [(u, v) for u in range(3) for v in range(3) if u != v]
    for mask in range(1 << 6):
        e = np.array([p for i, p in enumerate(pairs) if mask >> i & 1], np.int64).reshape(-1, 2)
        for fill in (0.0, 1.0):
            g = orc.build_csr(3, e[:, 0], e[:, 1], None, False, fill)
            check_canonical(g)
            np.testing.assert_array_equal(g.dense(), dense_adj(3, e[:, 0], e[:, 1], undirected=False, fill=fill))


def test_build_multigraph_weights_loops():
    """Duplicates, input self-loops, explicit zeros and weights (A2, A4, A5, A6)."""
    rng = np.random.default_rng(7)
    for trial in range(50):
        n = int(rng.integers(1, 30))
        m = int(rng.integers(0, 120))
        src = rng.integers(0, n, m)
        dst = rng.integers(0, n, m)
        w = rng.integers(0, 4, m).astype(np.float32)  # integer weights: sums exact
        und = bool(trial % 2)
        g = orc.build_csr(n, src, dst, w, und, 1.0)
        check_canonical(g)
        D = dense_adj(n, src, dst, w, und, 1.0)
        np.testing.assert_array_equal(g.dense(), D)
        # explicit zeros are kept as structure: every generated (row, col) appears
        pattern = np.zeros((n, n), bool)
        pattern[src, dst] = True
        if und:
            pattern[dst, src] = True
        pattern[np.arange(n), np.arange(n)] = True
        assert g.nnz == pattern.sum()


def test_build_fp64_coalesce_rounds_once():
    """Three fp32 weights whose fp32 running sum differs from the fp64 sum."""
    w = np.array([1.0, 2.0 ** -24, 2.0 ** -24], np.float32)
    g = orc.build_csr(2, [0, 0, 0], [1, 1, 1], w, False, 0.0)
    assert g.val[0] == np.float32(1.0 + 2.0 ** -23)  # fp32 sequential would give 1.0


def test_build_idempotent():
    s, d = chung_lu(500, 2000, seed=3)
    g = orc.build_csr(500, s, d, None, True, 1.0)
    rows = np.repeat(np.arange(500), np.diff(g.row_ptr))
    g2 = orc.build_csr(500, rows, g.col, g.val, False, 0.0)
    np.testing.assert_array_equal(g.row_ptr, g2.row_ptr)
    np.testing.assert_array_equal(g.col, g2.col)
    np.testing.assert_array_equal(g.val, g2.val)


def test_build_errors():
    with pytest.raises(orc.OracleError) as ei:
        orc.build_csr(3, [0], [3], None, True, 1.0)
    assert ei.value.code == -2
    with pytest.raises(orc.OracleError) as ei:
        orc.build_csr(3, [0], [1], [-1.0], True, 1.0)
    assert ei.value.code == -3
    with pytest.raises(orc.OracleError) as ei:
        orc.build_csr(3, [0], [1], [np.nan], True, 1.0)
    assert ei.value.code == -4


# ---------------------------------------------------------------------------
# 2. degree + symmetric normalisation (oracle.c §2)
# ---------------------------------------------------------------------------

def _norm_dense(n, edges, fill=1.0):
    e = np.array(edges, np.int64).reshape(-1, 2)
    g = orc.build_csr(n, e[:, 0], e[:, 1], None, True, fill)
    deg, a64, a32 = orc.sym_norm(g)
    return g, deg, a64, a32, g.dense(a64)


def test_sym_norm_spec_examples(golden):
    for case in golden["spec_examples"]["sym_norm"]:
        g, deg, a64, a32, _ = _norm_dense(case["n"], case["edges"])
        assert np.all(a64 == case["expect_all"]), case["cite"]


def test_sym_norm_closed_forms(golden):
    for case in golden["closed_forms"]["cases"]:
        g, deg, a64, a32, Ad = _norm_dense(case["n"], case["edges"])
        if "all" in case:
            assert np.all(a64 == case["all"]), case["name"]
        for r, c, v in case.get("entries", []):
            assert Ad[r, c] == v, (case["name"], r, c)


def test_sym_norm_kn():
    for n in (2, 3, 4, 7, 16, 33):
        edges = list(itertools.combinations(range(n), 2))
        _, deg, a64, a32, _ = _norm_dense(n, edges)
        assert np.all(deg == n) and np.all(a64 == 1.0 / n)


def test_sym_norm_vs_dense_and_spectrum():
    """Against the dense D^-1/2 A D^-1/2 product (different op order: 1e-15),
    symmetry, eigenvalues in [-1, 1], and the fp32 rounding of a64."""
    rng = np.random.default_rng(11)
    for trial in range(60):
        n = int(rng.integers(1, 33))
        m = int(rng.integers(0, n * (n - 1) // 2 + 1))
        s, d = erdos_renyi(n, m, seed=trial) if n > 1 else (np.zeros(0, np.int64), np.zeros(0, np.int64))
        w = weights(m, seed=trial) if trial % 3 == 0 else None
        g = orc.build_csr(n, s, d, w, True, 1.0)
        deg, a64, a32 = orc.sym_norm(g)
        Ad = g.dense(a64)
        Dn = dense_norm(dense_adj(n, s, d, w, True, 1.0 if w is None else 1.0))
        np.testing.assert_allclose(Ad, Dn, rtol=1e-14, atol=0)
        np.testing.assert_allclose(Ad, Ad.T, rtol=1e-15, atol=0)
        ev = np.linalg.eigvalsh(Ad)
        assert ev.min() >= -1 - 1e-12 and ev.max() <= 1 + 1e-12
        assert np.all(a32 == a64.astype(np.float32))
        np.testing.assert_array_equal(deg, g.dense().sum(1))


def test_sym_norm_zero_degree():
    """fill = 0 on an isolated node -> empty row; zero-weight edges -> a = 0 (A7)."""
    g = orc.build_csr(3, [0], [1], [0.0], True, 0.0)
    deg, a64, _ = orc.sym_norm(g)
    assert np.all(deg == 0) and np.all(a64 == 0) and g.row_ptr.tolist() == [0, 1, 2, 2]


# ---------------------------------------------------------------------------
# 3. SpMM (oracle.c §3)
# ---------------------------------------------------------------------------

def test_spmm_spec_examples(golden):
    for case in golden["spec_examples"]["gspmm_sum"]:
        h = np.array(case["h"], np.float32)
        y, cond = orc.spmm(case["row_ptr"], case["col"], None, h)
        np.testing.assert_array_equal(y, np.array(case["out"], np.float64)), case["cite"]


def test_spmm_vs_dense_500_random_graphs():
    """500 random graphs, n <= 64, F <= 16 vs dense A @ X; also
    cond == |A| @ |X| and |y| <= cond.  Catches transposed operand, wrong
    column, dropped term."""
    rng = np.random.default_rng(5)
    for t in range(500):
        n = int(rng.integers(1, 65))
        m = int(rng.integers(0, min(n * (n - 1) // 2, 4 * n) + 1))
        s, d = erdos_renyi(n, m, seed=t) if n > 1 else (np.zeros(0, np.int64), np.zeros(0, np.int64))
        und = t % 4 != 0
        if not und and m:
            d = rng.permutation(d)
        g = orc.build_csr(n, s, d, None, und, 1.0 if t % 5 else 0.0)
        _, a64, _ = orc.sym_norm(g)
        f = int(rng.integers(1, 17))
        x = uniform((n, f), seed=t)
        for a in (a64, None):
            y, cond = orc.spmm(g.row_ptr, g.col, a, x)
            Ad = g.dense(a64 if a is not None else np.ones(g.nnz))
            np.testing.assert_allclose(y, Ad @ x.astype(np.float64), rtol=1e-12, atol=1e-14)
            np.testing.assert_allclose(cond, np.abs(Ad) @ np.abs(x.astype(np.float64)), rtol=1e-12, atol=1e-14)
            assert np.all(np.abs(y) <= cond * (1 + 1e-12) + 1e-300)


def test_spmm_kn_column_means():
    n = 9
    e = np.array(list(itertools.combinations(range(n), 2)))
    g = orc.build_csr(n, e[:, 0], e[:, 1], None, True, 1.0)
    _, a64, _ = orc.sym_norm(g)
    x = uniform((n, 5), seed=1)
    y, _ = orc.spmm(g.row_ptr, g.col, a64, x)
    np.testing.assert_allclose(y, np.tile(x.astype(np.float64).mean(0), (n, 1)), rtol=1e-14)


@pytest.mark.parametrize("gen", ["chung_lu", "rmat"])
def test_spmm_identity_sqrt_degree(gen):
    """I1: A^ sqrt(d) = sqrt(d) exactly in real arithmetic (fp64 within 1e-13)
    on a power-law graph with hub rows; I2: A^ 1 = d^-1/2 * (A~ d^-1/2)."""
    n, m = 3000, 30000
    s, d = (chung_lu if gen == "chung_lu" else rmat)(n, m, seed=2)
    g = orc.build_csr(n, s, d, None, True, 1.0)
    deg, a64, _ = orc.sym_norm(g)
    x = np.sqrt(deg).astype(np.float32)[:, None]
    y, cond = orc.spmm(g.row_ptr, g.col, a64, x)
    # x is rounded to fp32, so compare against A^ applied to the rounded vector's
    # exact identity: sum_v a_uv sqrt(d_v) = sqrt(d_u); rounding of x costs <= 2^-24 rel
    np.testing.assert_allclose(y[:, 0], np.sqrt(deg), rtol=2e-7)
    y1, _ = orc.spmm(g.row_ptr, g.col, a64, np.ones((n, 1), np.float32))
    rows = np.repeat(np.arange(n), np.diff(g.row_ptr))
    i2 = np.bincount(rows, weights=g.val.astype(np.float64) / np.sqrt(deg[g.col]), minlength=n) / np.sqrt(deg)
    np.testing.assert_allclose(y1[:, 0], i2, rtol=1e-13)


def test_spmm_linearity_adjointness_permutation():
    n, m = 400, 3000
    s, d = chung_lu(n, m, seed=4)
    g = orc.build_csr(n, s, d, None, True, 1.0)
    _, a64, _ = orc.sym_norm(g)
    x1 = uniform((n, 3), seed=1)
    x2 = uniform((n, 3), seed=2)
    y1, _ = orc.spmm(g.row_ptr, g.col, a64, x1)
    y2, _ = orc.spmm(g.row_ptr, g.col, a64, x2)
    y12, _ = orc.spmm(g.row_ptr, g.col, a64, (x1 + x2))
    np.testing.assert_allclose(y12, y1 + y2, rtol=1e-6, atol=1e-6)  # x1+x2 rounded in fp32
    # adjointness <A x1, x2> = <x1, A x2> for symmetric A^
    assert abs((y1 * x2).sum() - (x1 * y2).sum()) < 1e-10
    # permutation equivariance: relabel nodes, Y permutes
    p = np.random.default_rng(0).permutation(n)
    gp = orc.build_csr(n, p[s], p[d], None, True, 1.0)
    _, ap, _ = orc.sym_norm(gp)
    xp = np.empty_like(x1)
    xp[p] = x1
    yp, _ = orc.spmm(gp.row_ptr, gp.col, ap, xp)
    np.testing.assert_allclose(yp[p], y1, rtol=1e-13, atol=1e-15)


def test_spmm_row_range():
    s, d = chung_lu(300, 1500, seed=6)
    g = orc.build_csr(300, s, d, None, True, 1.0)
    _, a64, _ = orc.sym_norm(g)
    x = features(300, 7)
    y, c = orc.spmm(g.row_ptr, g.col, a64, x)
    y2, c2 = orc.spmm(g.row_ptr, g.col, a64, x, r0=37, r1=211)
    np.testing.assert_array_equal(y[37:211], y2)
    np.testing.assert_array_equal(c[37:211], c2)


# ---------------------------------------------------------------------------
# 4-6. edge softmax, GAT scores, multi-head SpMM
# ---------------------------------------------------------------------------

def test_edge_softmax_spec_examples(golden):
    for case in golden["spec_examples"]["edge_softmax"]:
        lg = np.array(case["logits"])
        a = orc.edge_softmax([0, lg.size], lg, 1)
        np.testing.assert_allclose(a[:, 0], case["alpha"], atol=case["tol"], rtol=0), case["cite"]


def test_edge_softmax_vs_scipy_and_invariants():
    """Per-row scipy.special.softmax (library), rows sum to 1, shift invariance,
    no overflow at |logit| = 1e4, empty rows untouched."""
    s, d = chung_lu(700, 5000, seed=8)
    g = orc.build_csr(700, s, d, None, True, 0.0)
    H = 3
    lg = uniform((g.nnz, H), seed=9, low=-1e4, high=1e4).astype(np.float64)
    a = orc.edge_softmax(g.row_ptr, lg, H)
    assert np.all(np.isfinite(a))
    for u in range(700):
        b, e = g.row_ptr[u], g.row_ptr[u + 1]
        if b == e:
            continue
        np.testing.assert_allclose(a[b:e], scipy.special.softmax(lg[b:e], axis=0), rtol=1e-12, atol=1e-300)
        np.testing.assert_allclose(a[b:e].sum(0), 1.0, rtol=1e-13)
    a2 = orc.edge_softmax(g.row_ptr, lg + 123.0, H)
    np.testing.assert_allclose(a2, a, rtol=1e-9, atol=1e-300)


def test_gat_scores_pins(golden):
    """LeakyReLU special cases: slope 1 -> plain sum el[u] + er[v] (A13 indexing);
    slope 0 -> torch relu (library); S:253 example."""
    import torch
    s, d = chung_lu(200, 900, seed=3)
    g = orc.build_csr(200, s, d, None, True, 1.0)
    H = 4
    el = uniform((200, H), seed=1, low=-3, high=3)
    er = uniform((200, H), seed=2, low=-3, high=3)
    rows = np.repeat(np.arange(200), np.diff(g.row_ptr))
    lin = orc.gat_scores(g.row_ptr, g.col, el, er, H, slope=1.0)
    np.testing.assert_array_equal(lin, el[rows].astype(np.float64) + er[g.col].astype(np.float64))
    relu = orc.gat_scores(g.row_ptr, g.col, el, er, H, slope=0.0)
    np.testing.assert_array_equal(relu, torch.relu(torch.from_numpy(lin)).numpy())
    lr = orc.gat_scores(g.row_ptr, g.col, el, er, H, slope=0.2)
    np.testing.assert_allclose(lr, torch.nn.functional.leaky_relu(torch.from_numpy(lin), 0.2).numpy(), rtol=1e-15)
    ex = golden["spec_examples"]["leaky_relu"][0]
    v = orc.gat_scores([0, 1], [0], np.array([[ex["x"]]]), np.array([[0.0]]), 1, slope=ex["slope"])
    assert v[0, 0] == ex["y"]


def test_multihead_pins():
    """H = 1 equals spmm; zero head -> zeros; per-head dense
    matmul (library) for every head; uniform logits -> neighbourhood
    mean; constant Z per head -> constant (convexity)."""
    n = 500
    s, d = chung_lu(n, 3000, seed=12)
    g = orc.build_csr(n, s, d, None, True, 1.0)
    H, D = 4, 6
    z = uniform((n, H * D), seed=3)
    alpha = uniform((g.nnz, H), seed=4, low=0, high=1).astype(np.float64)
    alpha[:, 2] = 0.0
    y, cond = orc.multihead_spmm(g.row_ptr, g.col, alpha, z, H, D)
    for h in range(H):
        Ad = g.dense(alpha[:, h])
        np.testing.assert_allclose(y[:, h * D:(h + 1) * D], Ad @ z[:, h * D:(h + 1) * D].astype(np.float64),
                                   rtol=1e-12, atol=1e-14)
        ys, _ = orc.spmm(g.row_ptr, g.col, alpha[:, h], z[:, h * D:(h + 1) * D])
        np.testing.assert_array_equal(y[:, h * D:(h + 1) * D], ys)
    assert np.all(y[:, 2 * D:3 * D] == 0)
    # uniform logits -> mean over N(u) U {u}
    a_uni = orc.edge_softmax(g.row_ptr, np.zeros((g.nnz, H)), H)
    ym, _ = orc.multihead_spmm(g.row_ptr, g.col, a_uni, z, H, D)
    for u in (0, 17, 433):
        nb = g.col[g.row_ptr[u]:g.row_ptr[u + 1]]
        np.testing.assert_allclose(ym[u], z[nb].astype(np.float64).mean(0), rtol=1e-12, atol=1e-14)
    # convexity: constant per-head features give that constant
    zc = np.repeat(np.arange(1, H + 1, dtype=np.float32), D)[None, :].repeat(n, 0)
    sc = orc.gat_scores(g.row_ptr, g.col, uniform((n, H), 5, -3, 3), uniform((n, H), 6, -3, 3), H)
    yc, _ = orc.multihead_spmm(g.row_ptr, g.col, orc.edge_softmax(g.row_ptr, sc, H), zc, H, D)
    np.testing.assert_allclose(yc, zc, rtol=1e-13)


def test_attn_project_vs_einsum():
    n, H, D = 300, 8, 8
    z = uniform((n, H * D), seed=3)
    al = uniform((H, D), seed=4)
    ar = uniform((H, D), seed=5)
    el, er, elc, erc = orc.attn_project(z, al, ar, H, D)
    z3 = z.reshape(n, H, D).astype(np.float64)
    np.testing.assert_allclose(el, np.einsum("nhd,hd->nh", z3, al.astype(np.float64)), rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(er, np.einsum("nhd,hd->nh", z3, ar.astype(np.float64)), rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(elc, np.einsum("nhd,hd->nh", np.abs(z3), np.abs(al.astype(np.float64))), rtol=1e-12)


# ---------------------------------------------------------------------------
# 8-9. partition and slice
# ---------------------------------------------------------------------------

def test_partition_vs_searchsorted():
    for seed in range(5):
        n = 1000 + 500 * seed
        s, d = chung_lu(n, 8 * n, seed=seed)
        g = orc.build_csr(n, s, d, None, True, 1.0)
        for P in (1, 2, 3, 4, 8):
            b = orc.partition_rows(g.row_ptr, P)
            t = -(-np.arange(P + 1) * g.nnz // P)
            ref = np.searchsorted(g.row_ptr[:n], t, side="left")
            ref[0], ref[P] = 0, n
            np.testing.assert_array_equal(b, ref)
            assert np.all(np.diff(b) >= 0)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_slice_gathered_layout_equals_global(P):
    """T1: partition -> slice -> SpMM on the padded all-gather layout equals the
    unpartitioned oracle exactly (same fp64 ops in the same order)."""
    n = 1500
    s, d = chung_lu(n, 9000, seed=P)
    g = orc.build_csr(n, s, d, None, True, 1.0)
    _, a64, a32 = orc.sym_norm(g)
    x = features(n, 5)
    yg, _ = orc.spmm(g.row_ptr, g.col, a32.astype(np.float64), x)
    b = orc.partition_rows(g.row_ptr, P)
    npad = int(np.diff(b).max())
    xg = np.zeros((P * npad, 5), np.float32)
    for q in range(P):
        xg[q * npad:q * npad + b[q + 1] - b[q]] = x[b[q]:b[q + 1]]
    for r in range(P):
        rp, co, vo = orc.csr_slice(g.row_ptr, g.col, a32, b, r, npad)
        yl, _ = orc.spmm(rp, co, vo.astype(np.float64), xg)
        np.testing.assert_array_equal(yl, yg[b[r]:b[r + 1]])


# ---------------------------------------------------------------------------
# 3b. GSpMM reduce variants (oracle.c §3b, NEXT-2)
# ---------------------------------------------------------------------------

def test_gspmm_spec_example(golden):
    """row 0 -> {1,2}, h=[[1,2],[3,4],[5,6]]: sum [8,10], mean [4,5],
    max [5,6] (min [3,4] by the same hand evaluation); empty rows give zeros."""
    case = golden["spec_examples"]["gspmm_reduce"][0]
    h = np.array(case["h"], np.float32)
    for red in ("sum", "mean", "max", "min"):
        y = orc.gspmm(case["row_ptr"], case["col"], None, h, red)
        np.testing.assert_array_equal(y, np.array(case[red], np.float64), err_msg=red)


def test_gspmm_vs_dense_numpy():
    """Against NumPy reductions over each row's gathered rows (masked dense),
    with and without edge weights; sum equals orc.spmm exactly."""
    rng = np.random.default_rng(21)
    for t in range(60):
        n = int(rng.integers(1, 50))
        m = int(rng.integers(0, 3 * n + 1))
        src = rng.integers(0, n, m)
        dst = rng.integers(0, n, m)
        g = orc.build_csr(n, src, dst, None, bool(t % 2), 0.0 if t % 3 == 0 else 1.0)
        w = uniform(g.nnz, seed=t, low=-2, high=2).astype(np.float64) if t % 4 else None
        f = int(rng.integers(1, 9))
        x = uniform((n, f), seed=100 + t)
        for red in ("sum", "mean", "max", "min"):
            y = orc.gspmm(g.row_ptr, g.col, w, x, red)
            for u in range(n):
                b, e = g.row_ptr[u], g.row_ptr[u + 1]
                if b == e:
                    assert np.all(y[u] == 0)
                    continue
                vals = (w[b:e, None] if w is not None else 1.0) * x[g.col[b:e]].astype(np.float64)
                ref = {"sum": vals.sum(0), "mean": vals.mean(0), "max": vals.max(0), "min": vals.min(0)}[red]
                np.testing.assert_allclose(y[u], ref, rtol=1e-13, atol=1e-15, err_msg=red)
        ys, _ = orc.spmm(g.row_ptr, g.col, w, x)
        np.testing.assert_array_equal(orc.gspmm(g.row_ptr, g.col, w, x, "sum"), ys)


# ---------------------------------------------------------------------------
# 3c. K-step propagation (oracle.c §3c, NEXT-4)
# ---------------------------------------------------------------------------

def test_ppr_coeffs_spec_examples():
    """alpha=1,K=3 -> [1,0,0,0]; alpha=0.5,K=2 -> [0.5,0.25,0.125];
    sum = 1-(1-alpha)^(K+1)."""
    np.testing.assert_array_equal(orc.ppr_coeffs(1.0, 3), [1, 0, 0, 0])
    np.testing.assert_array_equal(orc.ppr_coeffs(0.5, 2), [0.5, 0.25, 0.125])
    th = orc.ppr_coeffs(0.1, 10)
    assert abs(th.sum() - (1 - 0.9 ** 11)) < 1e-15


def test_propagate_vs_dense_matrix_polynomial():
    """sum_k theta_k A^k X against numpy.linalg.matrix_power on small graphs;
    K = 0 gives theta_0 X; theta = e_1 gives the single SpMM."""
    rng = np.random.default_rng(31)
    for t in range(25):
        n = int(rng.integers(1, 40))
        m = int(rng.integers(0, 3 * n + 1))
        g = orc.build_csr(n, rng.integers(0, n, m), rng.integers(0, n, m), None, bool(t % 2), 1.0)
        _, a64, _ = orc.sym_norm(g)
        A = g.dense(a64)
        x = uniform((n, 4), seed=t)
        K = int(rng.integers(0, 6))
        th = uniform(K + 1, seed=50 + t).astype(np.float64)
        y, cond = orc.propagate(g.row_ptr, g.col, a64, x, th)
        ref = sum(th[k] * np.linalg.matrix_power(A, k) @ x.astype(np.float64) for k in range(K + 1))
        np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-13)
        assert np.all(np.abs(y) <= cond * (1 + 1e-12) + 1e-300)
    y1, _ = orc.propagate(g.row_ptr, g.col, a64, x, [0.0, 1.0])
    ys, _ = orc.spmm(g.row_ptr, g.col, a64, x)
    np.testing.assert_allclose(y1, ys, rtol=1e-15, atol=0)


def test_propagate_sqrt_degree_eigenvector():
    """A^ sqrt(d) = sqrt(d) => sum_k theta_k A^k sqrt(d) = (sum theta) sqrt(d)
    on a power-law graph (PPR coefficients)."""
    s, d = chung_lu(2000, 16000, seed=9)
    g = orc.build_csr(2000, s, d, None, True, 1.0)
    deg, a64, _ = orc.sym_norm(g)
    x = np.sqrt(deg).astype(np.float32)[:, None]
    th = orc.ppr_coeffs(0.1, 10)
    y, _ = orc.propagate(g.row_ptr, g.col, a64, x, th)
    np.testing.assert_allclose(y[:, 0], th.sum() * np.sqrt(deg), rtol=3e-7)


# ---------------------------------------------------------------------------
# 10. GAT backward pieces (oracle.c §10, NEXT-3)
# ---------------------------------------------------------------------------

def test_sddmm_spec_examples(golden):
    for case in golden["spec_examples"]["sddmm"]:
        e = np.array(case["edges"], np.int64).reshape(-1, 2)
        g = orc.build_csr(case["n"], e[:, 0], e[:, 1], None, False, 0.0)
        t = orc.sddmm(g.row_ptr, g.col, np.array(case["p"], np.float32), np.array(case["q"], np.float32))
        np.testing.assert_array_equal(t[:, 0], case["t"]), case["cite"]
    # self-loops only, p = q -> ||p[u]||^2
    p = uniform((7, 5), seed=3)
    g = orc.build_csr(7, [], [], None, False, 1.0)
    t = orc.sddmm(g.row_ptr, g.col, p, p)
    np.testing.assert_allclose(t[:, 0], (p.astype(np.float64) ** 2).sum(1), rtol=1e-15)


def test_sddmm_equals_masked_dense_product():
    """masking dense P Q^T by A's pattern equals sddmm (per head)."""
    s, d = chung_lu(300, 2000, seed=4)
    g = orc.build_csr(300, s, d, None, True, 1.0)
    H, D = 3, 5
    p = uniform((300, H * D), seed=5)
    q = uniform((300, H * D), seed=6)
    t = orc.sddmm(g.row_ptr, g.col, p, q, heads=H)
    rows = np.repeat(np.arange(300), np.diff(g.row_ptr))
    for h in range(H):
        PQ = p[:, h * D:(h + 1) * D].astype(np.float64) @ q[:, h * D:(h + 1) * D].astype(np.float64).T
        np.testing.assert_allclose(t[:, h], PQ[rows, g.col], rtol=1e-12, atol=1e-14)


def test_csr_transpose_vs_scipy():
    import scipy.sparse as sp
    rng = np.random.default_rng(8)
    for t in range(10):
        n, m = int(rng.integers(1, 60)), int(rng.integers(0, 300))
        g = orc.build_csr(n, rng.integers(0, n, m), rng.integers(0, n, m), None, False, 0.0)
        vals = np.arange(1, g.nnz + 1, dtype=np.float64)  # distinct values track the permutation
        rp, ct, pm = orc.csr_transpose(g.row_ptr, g.col, n)
        T = sp.csr_matrix((vals, g.col, g.row_ptr), shape=(n, n)).T.tocsr()
        T.sort_indices()
        np.testing.assert_array_equal(rp, T.indptr)
        np.testing.assert_array_equal(ct, T.indices)
        np.testing.assert_array_equal(vals[pm], T.data)
        rp2, ct2, pm2 = orc.csr_transpose(rp, ct, n)  # (A^T)^T = A
        np.testing.assert_array_equal(rp2, g.row_ptr)
        np.testing.assert_array_equal(ct2, g.col)
        np.testing.assert_array_equal(pm[pm2], np.arange(g.nnz))


def test_edge_softmax_backward_vs_dense_jacobian():
    """ds = J^T dalpha with the dense softmax Jacobian J = diag(a) - a a^T per row."""
    s, d = chung_lu(200, 900, seed=2)
    g = orc.build_csr(200, s, d, None, True, 1.0)
    H = 2
    lg = uniform((g.nnz, H), seed=3, low=-3, high=3).astype(np.float64)
    a = orc.edge_softmax(g.row_ptr, lg, H)
    da = uniform((g.nnz, H), seed=4).astype(np.float64)
    ds = orc.edge_softmax_backward(g.row_ptr, a, da, H)
    for u in range(0, 200, 7):
        b, e = g.row_ptr[u], g.row_ptr[u + 1]
        for h in range(H):
            al = a[b:e, h]
            J = np.diag(al) - np.outer(al, al)
            np.testing.assert_allclose(ds[b:e, h], J.T @ da[b:e, h], rtol=1e-12, atol=1e-15)


def test_gat_backward_vs_finite_differences():
    """Central differences of L = <dY, Y(el, er, z)> through the FORWARD oracle
    (gat_scores -> edge_softmax -> multihead_spmm).  Inputs are multiples of
    2^-6 and eps = 2^-12, so x +- eps is exact in fp32; the O(eps^2) remainder
    is far below the 1e-5 tolerance."""
    rng = np.random.default_rng(12)
    n, H, D = 40, 2, 3
    s, d = erdos_renyi(n, 120, seed=5)
    g = orc.build_csr(n, s, d, None, True, 1.0)
    q = lambda shape: (rng.integers(-128, 128, shape) / 64.0).astype(np.float32)
    el, er, z, dy = q((n, H)), q((n, H)), q((n, H * D)), q((n, H * D))

    def loss(el_, er_, z_):
        sc = orc.gat_scores(g.row_ptr, g.col, el_, er_, H, 0.2)
        al = orc.edge_softmax(g.row_ptr, sc, H)
        y, _ = orc.multihead_spmm(g.row_ptr, g.col, al, z_, H, D)
        return float((y * dy.astype(np.float64)).sum())

    dz, d_el, d_er, dt = orc.gat_backward(g.row_ptr, g.col, el, er, z, dy, H, D, 0.2)
    eps = 2.0 ** -12
    for arr, grad in ((el, d_el), (er, d_er), (z, dz)):
        for _ in range(12):
            i, j = int(rng.integers(0, arr.shape[0])), int(rng.integers(0, arr.shape[1]))
            orig = arr[i, j]
            arr[i, j] = orig + eps
            lp = loss(el, er, z)
            arr[i, j] = orig - eps
            lm = loss(el, er, z)
            arr[i, j] = orig
            fd = (lp - lm) / (2 * eps)
            assert abs(fd - grad[i, j]) <= 1e-5 * max(1.0, abs(fd)), (fd, grad[i, j])
    # d_el is the row sum and d_er the column sum of dt
    rows = np.repeat(np.arange(n), np.diff(g.row_ptr))
    np.testing.assert_allclose(d_el, np.stack([np.bincount(rows, dt[:, h], n) for h in range(H)], 1), rtol=1e-12)
    np.testing.assert_allclose(d_er, np.stack([np.bincount(g.col, dt[:, h], n) for h in range(H)], 1), rtol=1e-12)


def test_attn_project_backward_vs_finite_differences():
    """Central differences of L = <g_l, el> + <g_r, er> through orc.attn_project
    (linear: exact up to rounding) for z, a_l, a_r."""
    rng = np.random.default_rng(3)
    n, H, D = 30, 2, 4
    q = lambda shape: (rng.integers(-64, 64, shape) / 32.0).astype(np.float32)
    z, al, ar = q((n, H * D)), q((H, D)), q((H, D))
    gl, gr = rng.standard_normal((n, H)), rng.standard_normal((n, H))

    def loss(z_, al_, ar_):
        el, er, _, _ = orc.attn_project(z_, al_, ar_, H, D)
        return float((el * gl).sum() + (er * gr).sum())

    dz, d_al, d_ar = orc.attn_project_backward(z, al, ar, gl, gr, H, D)
    eps = 2.0 ** -10
    for arr, grad in ((z, dz), (al, d_al.reshape(H, D)), (ar, d_ar.reshape(H, D))):
        for _ in range(10):
            i, j = int(rng.integers(0, arr.shape[0])), int(rng.integers(0, arr.shape[1]))
            o = arr[i, j]
            arr[i, j] = o + eps
            lp = loss(z, al, ar)
            arr[i, j] = o - eps
            lm = loss(z, al, ar)
            arr[i, j] = o
            assert abs((lp - lm) / (2 * eps) - grad[i, j]) <= 1e-9 * max(1.0, abs(grad[i, j]))


# ---------------------------------------------------------------------------
# 11. inference layers (oracle.c §11, NEXT-1)
# ---------------------------------------------------------------------------

def test_linear_vs_numpy_and_activations():
    x = uniform((50, 17), seed=1)
    w = uniform((17, 9), seed=2)
    b = uniform(9, seed=3)
    y, cond = orc.linear(x, w, b)
    np.testing.assert_allclose(y, x.astype(np.float64) @ w.astype(np.float64) + b, rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(cond, np.abs(x.astype(np.float64)) @ np.abs(w.astype(np.float64)) + np.abs(b),
                               rtol=1e-13)
    import torch
    v = uniform((6, 7), seed=4, low=-3, high=3).astype(np.float64)
    np.testing.assert_array_equal(orc.bias_act(v, None, "relu"), torch.relu(torch.from_numpy(v)).numpy())
    np.testing.assert_allclose(orc.bias_act(v, None, "elu"), torch.nn.functional.elu(torch.from_numpy(v)).numpy(),
                               rtol=1e-15, atol=1e-300)


def test_gcn_layer_vs_dense_eq_gcn_layer():
    """Eq. gcn_layer: act(A^ X W + b) against dense NumPy; the SPEC
    example S:496 (K2, X=[[1],[0]], W=[1], A^ all 0.5 -> [[0.5],[0.5]])."""
    s, d = chung_lu(200, 800, seed=6)
    g = orc.build_csr(200, s, d, None, True, 1.0)
    _, a64, _ = orc.sym_norm(g)
    x = uniform((200, 12), seed=7)
    w = uniform((12, 5), seed=8)
    b = uniform(5, seed=9)
    for act in ("none", "relu", "elu"):
        y, _ = orc.gcn_layer(g.row_ptr, g.col, a64, x, w, b, act)
        ref = orc.bias_act(g.dense(a64) @ (x.astype(np.float64) @ w.astype(np.float64)), b, act)
        np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-13)
    g2 = orc.build_csr(2, [0], [1], None, True, 1.0)
    _, a2, _ = orc.sym_norm(g2)
    y2, _ = orc.gcn_layer(g2.row_ptr, g2.col, a2, np.array([[1.0], [0.0]], np.float32), np.array([[1.0]], np.float32),
                          None, "none")
    np.testing.assert_array_equal(y2, [[0.5], [0.5]])


# ---------------------------------------------------------------------------
# 12. tolerance scales (cond) -- every parity bound's scale is pinned against
#     an independent dense |.| evaluation, so an indexing slip that inflates
#     (or deflates) cond cannot silently change a parity bar
# ---------------------------------------------------------------------------

def _graph(n, m, seed, undirected=True):
    s, d = chung_lu(n, m, seed=seed)
    return orc.build_csr(n, s, d, None, undirected, 1.0)


def test_cond_multihead_equals_dense_abs():
    """orc_multihead_spmm's cond[u,h,:] == |A_h| @ |Z_h| per head (dense), with
    signed alpha (so |.| placement matters) and a zero head."""
    n = 400
    g = _graph(n, 2500, seed=21)
    for H, D in ((1, 3), (4, 6), (8, 2)):
        z = uniform((n, H * D), seed=3)
        alpha = uniform((g.nnz, H), seed=4, low=-1, high=1).astype(np.float64)
        alpha[:, H // 2] = 0.0
        _, cond = orc.multihead_spmm(g.row_ptr, g.col, alpha, z, H, D)
        for h in range(H):
            Ad = np.abs(g.dense(alpha[:, h]))
            np.testing.assert_allclose(cond[:, h * D:(h + 1) * D], Ad @ np.abs(z[:, h * D:(h + 1) * D].astype(np.float64)),
                                       rtol=1e-12, atol=0)
        assert np.all(cond[:, (H // 2) * D:(H // 2 + 1) * D] == 0)
        # row ranges give the same rows
        _, c2 = orc.multihead_spmm(g.row_ptr, g.col, alpha, z, H, D, r0=100, r1=180)
        np.testing.assert_array_equal(c2, cond[100:180])


def test_cond_spmm_row_range_and_dense():
    n = 300
    g = _graph(n, 2000, seed=22)
    _, a64, _ = orc.sym_norm(g)
    x = uniform((n, 7), seed=5)
    _, cond = orc.spmm(g.row_ptr, g.col, a64, x)
    np.testing.assert_allclose(cond, np.abs(g.dense(a64)) @ np.abs(x.astype(np.float64)), rtol=1e-12, atol=0)
    _, c2 = orc.spmm(g.row_ptr, g.col, a64, x, r0=37, r1=200)
    np.testing.assert_array_equal(c2, cond[37:200])


def test_cond_gcn_layer_equals_dense_abs():
    """orc_gcn_layer's cond == |A^| (|X| |W|) + |b| (dense), before the activation."""
    n = 250
    g = _graph(n, 1200, seed=23)
    _, a64, _ = orc.sym_norm(g)
    x = uniform((n, 11), seed=7)
    w = uniform((11, 6), seed=8)
    b = uniform(6, seed=9)
    ref = np.abs(g.dense(a64)) @ (np.abs(x.astype(np.float64)) @ np.abs(w.astype(np.float64))) + np.abs(b)
    for act in ("none", "relu", "elu"):
        _, cond = orc.gcn_layer(g.row_ptr, g.col, a64, x, w, b, act)
        np.testing.assert_allclose(cond, ref, rtol=1e-12, atol=0)
    _, c0 = orc.gcn_layer(g.row_ptr, g.col, a64, x, w, None, "relu")
    np.testing.assert_allclose(c0, ref - np.abs(b), rtol=1e-12, atol=1e-15)


def test_cond_attn_project_both_sides():
    """el_cond and er_cond == einsum over |z| |a_l| and |z| |a_r| respectively."""
    n, H, D = 200, 4, 5
    z = uniform((n, H * D), seed=3)
    al = uniform((H, D), seed=4)
    ar = uniform((H, D), seed=5) * 3.0  # different scale: a swapped cond would fail
    _, _, elc, erc = orc.attn_project(z, al, ar, H, D)
    z3 = np.abs(z.reshape(n, H, D).astype(np.float64))
    np.testing.assert_allclose(elc, np.einsum("nhd,hd->nh", z3, np.abs(al.astype(np.float64))), rtol=1e-12)
    np.testing.assert_allclose(erc, np.einsum("nhd,hd->nh", z3, np.abs(ar.astype(np.float64))), rtol=1e-12)


def test_cond_propagate_equals_matrix_power_of_abs():
    """orc_propagate's cond == sum_k |theta_k| |A|^k |X| (dense matrix powers),
    with signed thetas and signed weights."""
    rng = np.random.default_rng(77)
    for t in range(12):
        n = int(rng.integers(2, 40))
        m = int(rng.integers(1, 3 * n + 1))
        g = orc.build_csr(n, rng.integers(0, n, m), rng.integers(0, n, m), None, bool(t % 2), 1.0)
        _, a64, _ = orc.sym_norm(g)
        a = a64 * np.where(rng.random(g.nnz) < 0.3, -1.0, 1.0)  # signed weights
        A = np.abs(g.dense(a))
        x = uniform((n, 3), seed=t)
        K = int(rng.integers(1, 6))
        th = uniform(K + 1, seed=80 + t).astype(np.float64)
        _, cond = orc.propagate(g.row_ptr, g.col, a, x, th)
        ref = sum(abs(th[k]) * np.linalg.matrix_power(A, k) @ np.abs(x.astype(np.float64)) for k in range(K + 1))
        np.testing.assert_allclose(cond, ref, rtol=1e-12, atol=1e-300)


def test_omp_build_is_bit_identical():
    """liboracle_omp.so (the same oracle.c with -fopenmp, rows on all host
    cores) gives bit-identical y and cond: rows are independent and each row's
    arithmetic is unchanged."""
    n = 3000
    g = _graph(n, 30000, seed=31)
    _, a64, _ = orc.sym_norm(g)
    x = uniform((n, 37), seed=2)
    y1, c1 = orc.spmm(g.row_ptr, g.col, a64, x)
    y2, c2 = orc.spmm(g.row_ptr, g.col, a64, x, omp=True)
    np.testing.assert_array_equal(y1, y2)
    np.testing.assert_array_equal(c1, c2)
    al = uniform((g.nnz, 4), seed=3, low=0, high=1).astype(np.float64)
    z = uniform((n, 4 * 9), seed=4)
    m1 = orc.multihead_spmm(g.row_ptr, g.col, al, z, 4, 9)
    m2 = orc.multihead_spmm(g.row_ptr, g.col, al, z, 4, 9, omp=True, r0=5, r1=2900)
    np.testing.assert_array_equal(m1[0][5:2900], m2[0])
    np.testing.assert_array_equal(m1[1][5:2900], m2[1])
