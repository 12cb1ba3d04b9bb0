"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle.

Bars:
  * CSR structure (row_ptr, col) and A~ values: bit-exact.
  * normalised values and degrees: bit-exact (same IEEE-RN fp64 formula, A8).
  * Y (SpMM, multi-head, GAT): |y - y_ref| <= 1e-5 * cond + 1e-6 per element,
    cond = sum_e |a_e x_e| from the oracle (BASELINE.json north_star).
  * alpha: |a - a_ref| <= 1e-5 * a_ref + 1e-9; non-empty rows sum to 1 +- 1e-5.
  * el/er: |el - el_ref| <= 1e-5 * sum_d |a z| + 1e-6.
"""
import numpy as np
import pytest
import torch

import oracle as orc
import paper_2103_00959_b200 as G
from synth import CONFIGS, chung_lu, erdos_renyi, features, rmat, uniform, weights

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def assert_within(y, yref, cond, rel=1e-5, abs_=1e-6, what=""):
    y = np.asarray(y, np.float64)
    err = np.abs(y - yref)
    bound = rel * cond + abs_
    bad = ~(err <= bound)
    if bad.any():
        i = np.unravel_index(np.argmax(np.where(bad, err / bound, 0)), err.shape)
        raise AssertionError(f"{what}: {bad.sum()} / {err.size} elements out of bound; worst at {i}: "
                             f"y={y[i]} ref={yref[i]} err={err[i]:.3e} bound={bound[i]:.3e}")


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(DEV)


def host(t):
    return t.detach().cpu().numpy()


def gpu_build(n, src, dst, w=None, undirected=True, fill=1.0, idx=torch.int64):
    return G.gsp_coo_to_csr(n, dev(np.asarray(src, np.int64), idx), dev(np.asarray(dst, np.int64), idx),
                            None if w is None else dev(np.asarray(w, np.float32)), undirected, fill)


def graphs_small():
    """Adversarial small graphs: (name, n, src, dst, w, undirected, fill)."""
    rng = np.random.default_rng(0)
    out = [("n1-empty", 1, [], [], None, True, 1.0), ("n3-nofill-empty", 3, [], [], None, True, 0.0),
           ("k2", 2, [0], [1], None, True, 1.0), ("isolated-nofill", 6, [0, 1], [1, 2], None, True, 0.0)]
    for t in range(6):
        n = int(rng.integers(2, 80))
        m = int(rng.integers(0, 4 * n))
        src = rng.integers(0, n, m)
        dst = rng.integers(0, n, m)  # duplicates + self-loops in the input
        w = rng.integers(0, 4, m).astype(np.float32) if t % 2 else None
        out.append((f"multi{t}", n, src, dst, w, bool(t % 3), 1.0 if t != 4 else 0.0))
    s, d = erdos_renyi(300, 2000, seed=3)
    out.append(("er300-weighted", 300, s, d, weights(2000, seed=1), True, 1.0))
    s, d = chung_lu(4000, 30000, seed=2)
    out.append(("cl4000", 4000, s, d, None, True, 1.0))
    s, d = rmat(3000, 25000, seed=4)
    out.append(("rmat3000", 3000, s, d, None, True, 1.0))
    # hub rows around the CTA-cooperative threshold and a big star
    hub_deg = [1, 31, 32, 33, 511, 512, 513, 1024, 5000]
    src, dst = [], []
    base = len(hub_deg)
    for i, dg in enumerate(hub_deg):
        src += [i] * dg
        dst += list(range(base, base + dg))
        base += dg
    out.append(("hubs", base, src, dst, None, False, 1.0))
    # many long rows (row statistics' long CTAs: several per 128-row slice,
    # more than a group's slots, lengths at and around tile multiples for
    # every head count) among short ones, directed
    rng2 = np.random.default_rng(11)
    nl = 2000
    degs = np.where(rng2.random(nl) < 0.3, rng2.integers(30, 1300, nl), rng2.integers(0, 20, nl))
    degs[:40] = [31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 256, 257, 511, 512, 513, 1023, 1024, 1025,
                 2047, 2048, 2049, 200, 300, 400, 500, 600, 700, 800, 900, 1000, 1100, 1200, 130, 140, 150,
                 160, 170, 180, 190, 1]
    src = np.repeat(np.arange(nl), degs)
    dst = rng2.integers(0, nl, src.size)
    out.append(("longrows", nl, src, dst, None, False, 1.0))
    out.append(("star100k", 100001, [0] * 100000, list(range(1, 100001)), None, True, 1.0))
    return out


SMALL = graphs_small()


@pytest.fixture(scope="module")
def built():
    """name -> (oracle CSR, gpu CSR, (deg, a64, a32) oracle, gpu normalised CSR)"""
    res = {}
    for name, n, s, d, w, und, fill in SMALL:
        go = orc.build_csr(n, s, d, w, und, fill)
        gg = gpu_build(n, s, d, w, und, fill)
        no = orc.sym_norm(go)
        gn = G.gsp_sym_normalize(gg)
        res[name] = (go, gg, no, gn)
    return res


# ---------------------------------------------------------------- a1, a2

def test_build_bit_exact(built):
    for name, (go, gg, _, _) in built.items():
        assert gg.nnz == go.nnz, name
        np.testing.assert_array_equal(host(gg.row_ptr), go.row_ptr, err_msg=name)
        np.testing.assert_array_equal(host(gg.col), go.col, err_msg=name)
        np.testing.assert_array_equal(host(gg.val).view(np.uint32), go.val.view(np.uint32), err_msg=name)


@pytest.mark.parametrize("idx", [torch.int32, torch.int64])
def test_build_index_types_and_brute_force(idx):
    import itertools
    n = 5
    pairs = list(itertools.combinations(range(n), 2))
    for mask in range(0, 1 << len(pairs), 7):
        e = np.array([p for i, p in enumerate(pairs) if mask >> i & 1], np.int64).reshape(-1, 2)
        go = orc.build_csr(n, e[:, 0], e[:, 1], None, True, 1.0)
        gg = gpu_build(n, e[:, 0], e[:, 1], None, True, 1.0, idx=idx)
        np.testing.assert_array_equal(host(gg.row_ptr), go.row_ptr)
        np.testing.assert_array_equal(host(gg.col), go.col)
        np.testing.assert_array_equal(host(gg.val), go.val)


def test_build_errors():
    with pytest.raises(G.GspError) as ei:
        gpu_build(5, [0, 1], [1, 5])
    assert ei.value.status == 2
    with pytest.raises(G.GspError) as ei:
        gpu_build(5, [0, 1], [1, 2], w=[1.0, -1.0])
    assert ei.value.status == 3
    with pytest.raises(G.GspError) as ei:
        gpu_build(5, [0, 1], [1, 2], w=[np.inf, 1.0])
    assert ei.value.status == 4


def test_normalize_bit_exact(built):
    for name, (go, gg, (deg, a64, a32), gn) in built.items():
        np.testing.assert_array_equal(host(gn.deg), deg, err_msg=name)
        np.testing.assert_array_equal(host(gn.val).view(np.uint32), a32.view(np.uint32), err_msg=name)


def test_normalize_in_place(built):
    go, gg, (deg, a64, a32), _ = built["cl4000"]
    g2 = G.CSR(gg.row_ptr, gg.col, gg.val.clone(), gg.n_cols)
    gn = G.gsp_sym_normalize(g2, in_place=True)
    assert gn.val.data_ptr() == g2.val.data_ptr()
    np.testing.assert_array_equal(host(gn.val), a32)


# ---------------------------------------------------------------- a3

FS = [1, 2, 3, 4, 5, 31, 32, 33, 127, 128, 129, 602, 1433]



@pytest.mark.parametrize("kind", ["halves", "thirds", "eight", "empty-first", "single"])
def test_colblock_structure_and_spmm(built, kind):
    """Column blocks (gsp.h): every block is exactly the entries of A in its
    column range, in A's order (bit-exact), and the blocked SpMM is within the
    SpMM bound of the oracle and bitwise reproducible."""
    for name in ("multi1", "er300-weighted", "cl4000", "rmat3000", "hubs", "longrows"):
        go, gg, (deg, a64, a32), gn = built[name]
        n = go.n
        cuts = {"halves": [n // 2], "thirds": [n // 3, 2 * n // 3], "eight": [n * i // 8 for i in range(1, 8)],
                "empty-first": [0, n // 2], "single": []}[kind]
        bounds = [0] + cuts + [n]
        blocks = G.gsp_csr_colblock(gn, bounds)
        rows = np.repeat(np.arange(n), np.diff(go.row_ptr))
        for k in range(len(bounds) - 1):
            m = (go.col >= bounds[k]) & (go.col < bounds[k + 1])
            rp = np.zeros(n + 1, np.int64)
            rp[1:] = np.cumsum(np.bincount(rows[m], minlength=n))
            b = blocks.block(k)
            assert np.array_equal(host(b.row_ptr), rp), (name, kind, k)
            assert np.array_equal(host(b.col), go.col[m]), (name, kind, k)
            assert np.array_equal(host(b.val), a32[m]), (name, kind, k)
        for f in (1, 33, 128, 300):
            x = features(n, f, f, seed=f)
            yref, cond = orc.spmm(go.row_ptr, go.col, a64, x, f=f)
            y1 = G.gsp_spmm_blocked(blocks, dev(x), f=f)
            y2 = G.gsp_spmm_blocked(blocks, dev(x), f=f)
            assert torch.equal(y1, y2)
            assert_within(host(y1)[:, :f], yref, cond, what=f"{name} {kind} f={f}")


@pytest.mark.parametrize("f", FS)
def test_spmm_parity(built, f):
    for name in ("k2", "isolated-nofill", "multi1", "multi4", "er300-weighted", "cl4000", "rmat3000", "hubs"):
        go, gg, (deg, a64, a32), gn = built[name]
        n = go.n
        for ld in sorted({f, (f + 3) // 4 * 4}):
            x = features(n, f, ld, seed=f)
            yref, cond = orc.spmm(go.row_ptr, go.col, a64, x, f=f)
            y = G.gsp_spmm(gn, dev(x), f=f)
            assert_within(host(y), yref, cond, what=f"{name} f={f} ld={ld}")
            # psi = copy (val == NULL): unit weights
            yref1, cond1 = orc.spmm(go.row_ptr, go.col, None, x, f=f)
            y1 = G.gsp_spmm(gn.with_val(None), dev(x), f=f)
            assert_within(host(y1), yref1, cond1, what=f"{name} unweighted f={f}")


@pytest.mark.parametrize("f", FS)
def test_spmm_f16_parity(built, f):
    """gsp_spmm_f16 (fp16 feature storage, fp32 arithmetic) vs the oracle run
    on the same fp16 values: the fp32 bound holds exactly as for gsp_spmm."""
    for name in ("k2", "isolated-nofill", "multi1", "er300-weighted", "cl4000", "rmat3000", "hubs"):
        go, gg, (deg, a64, a32), gn = built[name]
        n = go.n
        for ld in sorted({f, (f + 3) // 4 * 4, (f + 7) // 8 * 8}):
            xh = features(n, f, ld, seed=f).astype(np.float16)
            yref, cond = orc.spmm(go.row_ptr, go.col, a64, xh.astype(np.float64), f=f)
            y = G.gsp_spmm_f16(gn, torch.from_numpy(xh).to(DEV), f=f)
            assert_within(host(y), yref, cond, what=f"f16 {name} f={f} ld={ld}")
            y1 = G.gsp_spmm_f16(gn.with_val(None), torch.from_numpy(xh).to(DEV), f=f)
            yref1, cond1 = orc.spmm(go.row_ptr, go.col, None, xh.astype(np.float64), f=f)
            assert_within(host(y1), yref1, cond1, what=f"f16 {name} unweighted f={f}")


def test_spmm_unaligned_and_strided(built):
    go, gg, (deg, a64, a32), gn = built["cl4000"]
    n = go.n
    f = 37
    big = features(n, 40, 41, seed=9)  # ld = 41 (odd), base offset 1 float
    xt = dev(big)[:, 1:1 + f]
    yref, cond = orc.spmm(go.row_ptr, go.col, a64, big[:, 1:1 + f].copy(), f=f)
    yfull = torch.full((n, 50), 7.0, device=DEV)
    y = yfull[:, 3:3 + f]
    G.gsp_spmm(gn, xt, f=f, y=y)
    assert_within(host(y), yref, cond, what="unaligned")
    # padding columns untouched
    assert torch.all(yfull[:, :3] == 7.0) and torch.all(yfull[:, 3 + f:] == 7.0)


def test_spmm_hub_rows_and_star(built):
    for name in ("hubs", "star100k"):
        go, gg, (deg, a64, a32), gn = built[name]
        x = features(go.n, 64, seed=4)
        yref, cond = orc.spmm(go.row_ptr, go.col, a64, x)
        assert_within(host(G.gsp_spmm(gn, dev(x))), yref, cond, what=name)


@pytest.mark.parametrize("f", [256, 300])
def test_spmm_deterministic_and_config_invariant(built, f):
    """Bitwise identical for every slab width / block size (incl. the 256-col
    two-float4 path and the narrow tail launch: F=300 -> 2x128 + 64)."""
    go, gg, _, gn = built["rmat3000"]
    x = dev(features(go.n, f, seed=5))
    y0 = G.gsp_spmm(gn, x)
    if f == 300:
        assert G.gsp_spmm_plan_info(gn, x) == (2, 128, 64)
    for slab, blk in [(0, 0), (4, 0), (32, 512), (64, 300), (128, 10000), (8, 0), (16, 64), (256, 0), (256, 777)]:
        if slab == 256 and f % 8:  # two float4 per lane need ldx % 8 == 0 (gsp.h)
            with pytest.raises(G.GspError):
                G.gsp_spmm(gn, x, slab_cols=slab, block_nnz=blk)
            xp = torch.zeros((go.n, 304), device=DEV)
            xp[:, :f] = x
            y = G.gsp_spmm(gn, xp, f=f, slab_cols=slab, block_nnz=blk)
        else:
            y = G.gsp_spmm(gn, x, slab_cols=slab, block_nnz=blk)
        assert torch.equal(y, y0), (slab, blk)
    assert torch.equal(G.gsp_spmm(gn, x), y0)


def test_spmm_identity_sqrt_degree_full_c2():
    cfg = CONFIGS["C2"]
    s, d = chung_lu(cfg.n, cfg.m, seed=1)
    gn = G.gsp_sym_normalize(gpu_build(cfg.n, s, d))
    x = torch.sqrt(gn.deg).float()[:, None].contiguous()
    y = G.gsp_spmm(gn, x)
    np.testing.assert_allclose(host(y)[:, 0], np.sqrt(host(gn.deg)), rtol=2e-6)


def test_spmm_errors(built):
    _, _, _, gn = built["cl4000"]
    x = torch.zeros((gn.n_cols, 8), device=DEV)
    with pytest.raises(G.GspError) as ei:
        G.gsp_spmm(gn, x, y=x)
    assert ei.value.status == 5


# ---------------------------------------------------------------- a4 - a7

@pytest.mark.parametrize("H", [1, 2, 3, 4, 8, 16, 32])
def test_edge_softmax_parity(built, H):
    for name in ("multi0", "cl4000", "hubs", "longrows", "star100k"):
        go, gg, _, _ = built[name]
        for lo, hi in [(-3, 3), (-1e4, 1e4)]:
            lg = uniform((go.nnz, H), seed=H, low=lo, high=hi)
            aref = orc.edge_softmax(go.row_ptr, lg.astype(np.float64), H)
            a = host(G.gsp_edge_softmax(gg, dev(lg), H))
            assert np.all(np.isfinite(a))
            err = np.abs(a - aref)
            assert np.all(err <= 1e-5 * aref + 1e-9), (name, H, lo, err.max())
            rows = np.repeat(np.arange(go.n), np.diff(go.row_ptr))
            sums = np.zeros((go.n, H))
            np.add.at(sums, rows, a.astype(np.float64))
            nonempty = np.diff(go.row_ptr) > 0
            assert np.all(np.abs(sums[nonempty] - 1) <= 1e-5)
    # in place
    go, gg, _, _ = built["cl4000"]
    lg = uniform((go.nnz, H), seed=1)
    t = dev(lg)
    G.gsp_edge_softmax(gg, t, H, alpha=t)
    aref = orc.edge_softmax(go.row_ptr, lg.astype(np.float64), H)
    assert np.all(np.abs(host(t) - aref) <= 1e-5 * aref + 1e-9)


@pytest.mark.parametrize("H,D", [(1, 64), (2, 3), (4, 8), (8, 8), (8, 64), (3, 16), (2, 128), (4, 32), (16, 64), (1, 256), (5, 4)])
def test_attn_project_parity(H, D):
    n = 5000
    z = uniform((n, H * D), seed=3)
    al = uniform((H, D), seed=4)
    ar = uniform((H, D), seed=5)
    el_ref, er_ref, elc, erc = orc.attn_project(z, al, ar, H, D)
    el, er = G.gsp_attn_project(dev(z), dev(al.reshape(-1)), dev(ar.reshape(-1)), H, D)
    assert_within(host(el), el_ref, elc, what="el")
    assert_within(host(er), er_ref, erc, what="er")


@pytest.mark.parametrize("H,D", [(1, 1), (1, 64), (2, 3), (4, 8), (8, 8), (8, 64), (3, 16), (2, 64), (4, 32), (4, 1)])
def test_multihead_spmm_parity(built, H, D):
    for name in ("multi2", "cl4000", "hubs"):
        go, gg, _, _ = built[name]
        z = uniform((go.n, H * D), seed=3)
        alpha = uniform((go.nnz, H), seed=4, low=0, high=1)
        yref, cond = orc.multihead_spmm(go.row_ptr, go.col, alpha.astype(np.float64), z, H, D)
        y = G.gsp_multihead_spmm(gg, dev(alpha), dev(z), H, D)
        assert_within(host(y), yref, cond, what=f"{name} H={H} D={D}")


def _gat_ref(go, el, er, z, H, D, slope):
    s = orc.gat_scores(go.row_ptr, go.col, el, er, H, slope)
    a = orc.edge_softmax(go.row_ptr, s, H)
    y, cond = orc.multihead_spmm(go.row_ptr, go.col, a, z, H, D)
    return y, cond, a


@pytest.mark.parametrize("sched", ["staged", "stats-launch", "single-launch"])
@pytest.mark.parametrize("H,D", [(1, 64), (2, 3), (4, 8), (8, 8), (8, 64), (3, 16), (2, 64), (4, 32), (4, 1), (2, 256)])
def test_gat_aggregate_parity(built, H, D, sched):
    """The three schedules of gsp_gat_aggregate against the fp64 oracle:
    staged (statistics launch writes alpha head-major, the aggregate stages it
    with the CSR window), stats-launch ((m, 1/S) only, alpha formed in the
    aggregate; the schedule that also writes alpha_out) and single-launch
    (statistics reduced inside the aggregate)."""
    for name in ("multi0", "cl4000", "rmat3000", "hubs", "longrows"):
        go, gg, _, _ = built[name]
        n = go.n
        z = uniform((n, H * D), seed=3)
        for lo, hi in [(-3, 3), (-1e4, 1e4)]:
            el = uniform((n, H), seed=4, low=lo, high=hi)
            er = uniform((n, H), seed=5, low=lo, high=hi)
            yref, cond, aref = _gat_ref(go, el, er, z, H, D, 0.2)
            what = f"{name} H={H} D={D} range={hi} {sched}"
            if sched == "staged":
                y = G.gsp_gat_aggregate(gg, dev(el), dev(er), dev(z), H, D, 0.2)
                assert_within(host(y), yref, cond, what=what)
                continue
            y, a = G.gsp_gat_aggregate(gg, dev(el), dev(er), dev(z), H, D, 0.2, alpha_out=True,
                                       single_launch=sched == "single-launch")
            assert_within(host(y), yref, cond, what=what)
            err = np.abs(host(a) - aref)
            assert np.all(err <= 1e-5 * aref + 1e-9), (name, H, D, err.max())


def test_gat_uniform_scores_give_mean(built):
    go, gg, _, _ = built["cl4000"]
    H, D = 4, 8
    z = uniform((go.n, H * D), seed=3)
    zero = torch.zeros((go.n, H), device=DEV)
    y = host(G.gsp_gat_aggregate(gg, zero, zero, dev(z), H, D))
    for u in (0, 5, 77, 1234):
        nb = go.col[go.row_ptr[u]:go.row_ptr[u + 1]]
        np.testing.assert_allclose(y[u], z[nb].astype(np.float64).mean(0), rtol=1e-5, atol=1e-6)


# ---------------------------------------------------------------- multi-GPU partition

@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_partition_slice_bit_exact_and_invariant(built, P):
    go, gg, (deg, a64, a32), gn = built["rmat3000"]
    bref = orc.partition_rows(go.row_ptr, P)
    b, bdev = G.gsp_partition_rows(gn, P)
    np.testing.assert_array_equal(np.array(b), bref)
    np.testing.assert_array_equal(host(bdev), bref)
    npad = int(np.diff(bref).max())
    f = 96
    x = features(go.n, f, seed=8)
    y_global = host(G.gsp_spmm(gn, dev(x)))
    xg = np.zeros((P * npad, f), np.float32)
    for q in range(P):
        xg[q * npad:q * npad + bref[q + 1] - bref[q]] = x[bref[q]:bref[q + 1]]
    for r in range(P):
        rp, co, vo = orc.csr_slice(go.row_ptr, go.col, a32, bref, r, npad)
        sl = G.gsp_csr_slice(gn, b, r, npad)
        np.testing.assert_array_equal(host(sl.row_ptr), rp)
        np.testing.assert_array_equal(host(sl.col), co)
        np.testing.assert_array_equal(host(sl.val), vo)
        yl = host(G.gsp_spmm(sl, dev(xg)))
        # partition invariance: bitwise equal to the single-GPU result
        np.testing.assert_array_equal(yl, y_global[bref[r]:bref[r + 1]])


# ---------------------------------------------------------------- NEXT-2: GSpMM reduce variants

@pytest.mark.parametrize("reduce", ["sum", "mean", "max", "min"])
@pytest.mark.parametrize("f", [1, 5, 33, 128, 300])
def test_gspmm_reduce_parity(built, reduce, f):
    """max / min are exact (monotone rounding of exact products) -> bit-equal to
    the oracle on the same fp32 weights; sum / mean within 1e-5*cond(/deg)+1e-6."""
    for name in ("isolated-nofill", "multi1", "multi4", "er300-weighted", "cl4000", "hubs", "star100k"):
        go, gg, (deg, a64, a32), gn = built[name]
        x = features(go.n, f, (f + 3) // 4 * 4, seed=f + 11)
        for g, a in ((gn, a32.astype(np.float64)), (gn.with_val(None), None)):
            y = host(G.gsp_gspmm(g, dev(x), reduce, f=f))
            yref = orc.gspmm(go.row_ptr, go.col, a, x, reduce, f=f)
            if reduce in ("max", "min"):
                np.testing.assert_array_equal(y, yref.astype(np.float32), err_msg=f"{name} {reduce} f={f}")
            else:
                _, cond = orc.spmm(go.row_ptr, go.col, a, x, f=f)
                if reduce == "mean":
                    cnt = np.maximum(np.diff(go.row_ptr), 1)[:, None]
                    cond = cond / cnt
                assert_within(y, yref, cond, what=f"{name} {reduce} f={f}")


def test_gspmm_sum_equals_spmm_bitwise(built):
    go, gg, _, gn = built["rmat3000"]
    x = dev(features(go.n, 300, seed=3))
    assert torch.equal(G.gsp_gspmm(gn, x, "sum"), G.gsp_spmm(gn, x))


# ---------------------------------------------------------------- NEXT-4: K-step propagation

@pytest.mark.parametrize("K", [1, 2, 3, 10])
@pytest.mark.parametrize("f", [1, 41, 128, 300])
def test_propagate_parity(built, K, f):
    """y = sum_k theta_k A^k x (PPR coefficients) vs the fp64 oracle; the error
    of each of the K SpMMs is propagated by A, bound K*1e-5*cond + 1e-6."""
    th = orc.ppr_coeffs(0.1, K)
    for name in ("isolated-nofill", "multi0", "er300-weighted", "cl4000", "hubs"):
        go, gg, (deg, a64, a32), gn = built[name]
        x = features(go.n, f, (f + 3) // 4 * 4, seed=K + f)
        yref, cond = orc.propagate(go.row_ptr, go.col, a64, x, th, f=f)
        y = host(G.gsp_propagate(gn, dev(x), th, f=f))
        assert_within(y, yref, cond, rel=K * 1e-5, what=f"{name} K={K} f={f}")


def test_propagate_accumulate_step_semantics(built):
    """gsp_spmm_accumulate: t = A x, acc = c*t + s*src (or + acc)."""
    go, gg, _, gn = built["cl4000"]
    x = dev(features(go.n, 64, seed=1))
    src = dev(features(go.n, 64, seed=2))
    t = torch.empty_like(x)
    acc = torch.empty_like(x)
    G.gsp_spmm_accumulate(gn, x, acc, 0.5, t=t, src=src, src_coef=2.0)
    ax = G.gsp_spmm(gn, x)
    assert torch.equal(t, ax)
    assert torch.equal(acc, torch.addcmul(src * 2.0, ax, torch.tensor(0.5, device=DEV)))
    acc2 = acc.clone()
    G.gsp_spmm_accumulate(gn, x, acc2, -1.0)
    assert torch.equal(acc2, torch.addcmul(acc, ax, torch.tensor(-1.0, device=DEV)))


# ---------------------------------------------------------------- NEXT-3: GAT backward

def test_csr_transpose_bit_exact(built):
    for name in ("n1-empty", "isolated-nofill", "multi0", "multi4", "cl4000", "rmat3000", "hubs", "star100k"):
        go, gg, _, _ = built[name]
        rp, ct, pm = orc.csr_transpose(go.row_ptr, go.col, go.n)
        at, perm = G.gsp_csr_transpose(gg)
        np.testing.assert_array_equal(host(at.row_ptr), rp, err_msg=name)
        np.testing.assert_array_equal(host(at.col), ct, err_msg=name)
        np.testing.assert_array_equal(host(perm).astype(np.int64), pm, err_msg=name)


@pytest.mark.parametrize("H,D", [(1, 1), (1, 64), (2, 3), (4, 8), (8, 64), (3, 16), (1, 602), (8, 32), (4, 64), (2, 128), (16, 8)])
def test_sddmm_parity(built, H, D):
    """|t - t_ref| <= 1e-5 * sum_k |p q| + 1e-6 (D-term dot products)."""
    for name in ("multi1", "cl4000", "hubs"):
        go, gg, _, _ = built[name]
        p = uniform((go.n, H * D), seed=1)
        q = uniform((go.n, H * D), seed=2)
        tref = orc.sddmm(go.row_ptr, go.col, p, q, heads=H)
        cond = orc.sddmm(go.row_ptr, go.col, np.abs(p), np.abs(q), heads=H)
        t = host(G.gsp_sddmm(gg, dev(p), dev(q), heads=H))
        assert_within(t, tref, cond, what=f"{name} H={H} D={D}")


def test_edge_softmax_backward_parity(built):
    """|ds - ds_ref| <= 1e-5 * alpha (|dalpha| + sum_row alpha |dalpha|) + 1e-9."""
    for H in (1, 2, 4, 8):
        go, gg, _, _ = built["cl4000"]
        lg = uniform((go.nnz, H), seed=H, low=-3, high=3)
        a = G.gsp_edge_softmax(gg, dev(lg), H)
        da = uniform((go.nnz, H), seed=10 + H)
        ds = host(G.gsp_edge_softmax_backward(gg, a, dev(da), H))
        a64 = host(a).astype(np.float64)
        dsref = orc.edge_softmax_backward(go.row_ptr, a64, da.astype(np.float64), H)
        rows = np.repeat(np.arange(go.n), np.diff(go.row_ptr))
        rs = np.stack([np.bincount(rows, a64[:, h] * np.abs(da[:, h]), go.n) for h in range(H)], 1)
        cond = a64 * (np.abs(da) + rs[rows])
        assert_within(ds, dsref, cond, abs_=1e-9, what=f"H={H}")


@pytest.mark.parametrize("H,D", [(1, 64), (4, 8), (8, 64), (2, 3)])
def test_gat_aggregate_backward_parity(built, H, D):
    """dz, d_el, d_er vs the fp64 oracle.  Bounds from the arithmetic: dz is an
    A^T SpMM (1e-5 * sum alpha |dy|); dt = alpha (dalpha - <alpha, dalpha>)
    with dalpha an SDDMM, so |d dt| <= 1e-5 * alpha (c + sum_row alpha c),
    c = sddmm(|dy|, |z|); d_el / d_er sum those over rows / columns."""
    for name in ("multi0", "cl4000", "hubs"):
        go, gg, _, _ = built[name]
        n = go.n
        el = uniform((n, H), seed=4, low=-3, high=3)
        er = uniform((n, H), seed=5, low=-3, high=3)
        z = uniform((n, H * D), seed=6)
        dy = uniform((n, H * D), seed=7)
        at, perm = G.gsp_csr_transpose(gg)
        dz, d_el, d_er = [host(t) for t in G.gsp_gat_aggregate_backward(gg, at, perm, dev(el), dev(er), dev(z),
                                                                         dev(dy), H, D)]
        dz_r, del_r, der_r, dt_r = orc.gat_backward(go.row_ptr, go.col, el, er, z, dy, H, D)
        sc = orc.gat_scores(go.row_ptr, go.col, el, er, H)
        al = orc.edge_softmax(go.row_ptr, sc, H)
        rp_t, ct, pm = orc.csr_transpose(go.row_ptr, go.col, n)
        dz_c, _ = orc.multihead_spmm(rp_t, ct, al[pm], np.abs(dy), H, D)
        assert_within(dz, dz_r, dz_c, what=f"dz {name}")
        c = orc.sddmm(go.row_ptr, go.col, np.abs(dy), np.abs(z), heads=H)
        rows = np.repeat(np.arange(n), np.diff(go.row_ptr))
        rs = np.stack([np.bincount(rows, al[:, h] * c[:, h], n) for h in range(H)], 1)
        cdt = al * (c + rs[rows])
        cel = np.stack([np.bincount(rows, cdt[:, h], n) for h in range(H)], 1)
        cer = np.stack([np.bincount(go.col, cdt[:, h], n) for h in range(H)], 1)
        assert_within(d_el, del_r, cel, what=f"d_el {name}")
        assert_within(d_er, der_r, cer, what=f"d_er {name}")


def test_attn_project_backward_parity():
    n, H, D = 3000, 8, 64
    z = uniform((n, H * D), seed=1)
    al = uniform((H, D), seed=2)
    ar = uniform((H, D), seed=3)
    gl = uniform((n, H), seed=4)
    gr = uniform((n, H), seed=5)
    dz0 = uniform((n, H * D), seed=6)
    dz = dev(dz0)
    d_al, d_ar = G.gsp_attn_project_backward(dev(z), dev(al.reshape(-1)), dev(ar.reshape(-1)), dev(gl), dev(gr), dz,
                                             H, D)
    dz_r, dal_r, dar_r = orc.attn_project_backward(z, al, ar, gl, gr, H, D)
    _, dal_c, dar_c = orc.attn_project_backward(np.abs(z), al, ar, np.abs(gl), np.abs(gr), H, D)
    assert_within(host(d_al), dal_r, dal_c, what="d_al")
    assert_within(host(d_ar), dar_r, dar_c, what="d_ar")
    dzc, _, _ = orc.attn_project_backward(z, np.abs(al), np.abs(ar), np.abs(gl), np.abs(gr), H, D)
    assert_within(host(dz), dz0.astype(np.float64) + dz_r, np.abs(dz0) + dzc, what="dz")


# ---------------------------------------------------------------- NEXT-1: inference layers

def _lin_rel(f_in):
    """Bound for y = act(A (x W) + b): the GEMM bound (3xTF32 tensor cores,
    _tc_rel; it also covers an fp32 SGEMM's gamma_{f_in} <= f_in * 2^-24)
    followed by the SpMM bound 1e-5 (north_star); ReLU / ELU are 1-Lipschitz
    (DESIGN.md §7)."""
    return 1e-5 + _tc_rel(f_in)


def _tc_rel(f_in):
    """3xTF32 tensor-core GEMM bound: per product
    <= 2^-19 |x||w| (x_hi = the MMA's truncated read of x, the truncated lo
    parts and the dropped lo*lo term),
    plus f_in fp32 accumulations at <= 2u each (tensor-core accumulation is
    not assumed to round to nearest)."""
    return 2.0 ** -19 + f_in * 2.0 ** -23


@pytest.mark.parametrize("tc", [True, False], ids=["tcgen05", "cublas"])
@pytest.mark.parametrize("n,f_in,f_out", [(5000, 3, 5), (5000, 33, 7), (5000, 128, 41), (5000, 602, 128),
                                          (1, 1, 1), (128, 32, 16), (129, 31, 17), (3000, 1433, 256),
                                          (2000, 300, 128), (777, 500, 41), (1000, 64, 512), (500, 100, 300),
                                          (100, 512, 128), (129, 400, 16)])
def test_linear_parity(n, f_in, f_out, tc):
    # f_in >= 384 with f_out <= 128 takes the CTA-pair (shared W) kernel; odd
    # tile counts (777 -> 7, 100 -> 1, 129 -> 2 with a ragged tail) exercise
    # its padding CTA
    x = uniform((n, f_in), seed=1)
    w = uniform((f_in, f_out), seed=2)
    y = host(G.gsp_linear(dev(x), dev(w), tensor_cores=tc))
    yr, c = orc.linear(x, w)
    rel = _tc_rel(f_in) if tc else f_in * 2.0 ** -24 + 1e-7
    assert_within(y, yr, c, rel=rel, what=f"linear {n}x{f_in}x{f_out} tc={tc}")


@pytest.mark.parametrize("pattern", ["round_up", "round_down", "random_low_bits"])
def test_linear_tc_low_mantissa_bits(pattern):
    """X entries whose bits below TF32 precision decide how the tensor core
    reads them: with W = I every output is a single product x * 1, so the
    3xTF32 result must equal x to 2^-19 relative per element -- a truncating
    vs rounding misreading of x_hi would be off by up to 2^-10."""
    n, f = 256, 32
    rng = np.random.default_rng(7)
    mant = {"round_up": 3.0 * 2.0 ** -12, "round_down": 1.0 * 2.0 ** -12}
    if pattern in mant:
        x = np.full((n, f), 1.0 + mant[pattern], np.float32) * rng.choice([-1.0, 1.0], (n, f)).astype(np.float32)
    else:
        bits = rng.integers(0, 1 << 32, size=(n, f), dtype=np.uint64).astype(np.uint32)
        bits = (bits & np.uint32(0x807FFFFF)) | np.uint32(127 << 23)  # |x| in [1, 2), every mantissa bit random
        x = bits.view(np.float32)
    w = np.eye(f, dtype=np.float32)
    y = host(G.gsp_linear(dev(x), dev(w), tensor_cores=True)).astype(np.float64)
    err = np.abs(y - x.astype(np.float64)) / np.abs(x.astype(np.float64))
    assert err.max() <= 2.0 ** -19, f"{pattern}: max relative error {err.max():.3e}"


def test_linear_tc_padded_views():
    """Tensor-core GEMM on a padded X view (ld > f_in) into a padded Y view,
    and a graph-sized ragged tail (n % 128 != 0)."""
    n, f_in, f_out = 1001, 602, 128
    xb = torch.zeros((n, 604), device=DEV)
    x = uniform((n, f_in), seed=3)
    xb[:, :f_in] = dev(x)
    w = uniform((f_in, f_out), seed=4)
    yb = torch.full((n, 132), 7.0, device=DEV)
    G.gsp_linear(xb[:, :f_in], dev(w), y=yb[:, :f_out])
    yr, c = orc.linear(x, w)
    assert_within(host(yb[:, :f_out]), yr, c, rel=_tc_rel(f_in), what="padded")
    assert torch.all(yb[:, f_out:] == 7.0)  # padding columns untouched


@pytest.mark.parametrize("act", ["none", "relu", "elu"])
def test_gcn_layer_parity(built, act):
    for name in ("isolated-nofill", "cl4000", "hubs"):
        go, gg, (deg, a64, a32), gn = built[name]
        x = uniform((go.n, 37), seed=3)
        w = uniform((37, 20), seed=4)
        b = uniform(20, seed=5)
        y = host(G.gsp_gcn_layer(gn, dev(x), dev(w), dev(b), act))
        yr, c = orc.gcn_layer(go.row_ptr, go.col, a64, x, w, b, act)
        assert_within(y, yr, c, rel=_lin_rel(37), what=f"{name} {act}")


@pytest.mark.parametrize("single", [False, True], ids=["stats-launch", "single-launch"])
@pytest.mark.parametrize("H,D", [(4, 32), (1, 41), (8, 8)])
def test_gat_aggregate_bias_act_parity(built, H, D, single):
    go, gg, _, _ = built["cl4000"]
    n = go.n
    z = uniform((n, H * D), seed=3)
    el = uniform((n, H), seed=4, low=-3, high=3)
    er = uniform((n, H), seed=5, low=-3, high=3)
    b = uniform(H * D, seed=6)
    y = host(G.gsp_gat_aggregate_bias_act(gg, dev(el), dev(er), dev(z), H, D, dev(b), "elu", single_launch=single))
    s = orc.gat_scores(go.row_ptr, go.col, el, er, H)
    al = orc.edge_softmax(go.row_ptr, s, H)
    yr, c = orc.multihead_spmm(go.row_ptr, go.col, al, z, H, D)
    assert_within(y, orc.bias_act(yr, b, "elu"), c + np.abs(b), what=f"H={H} D={D}")


def test_gcn_inference_sampled_rows_c4():
    """2-layer GCN on C4 through paper_2103_00959_b200.inference: layer 1 vs the
    oracle on sampled rows; layer 2 from the GPU's own layer-1 output."""
    from paper_2103_00959_b200.inference import GCNParams, gcn_inference
    cfg = CONFIGS["C4"]
    from synth import graph_for
    s, d = graph_for(cfg, seed=1)
    gn = G.gsp_sym_normalize(gpu_build(cfg.n, s, d))
    go = orc.CSR(cfg.n, host(gn.row_ptr), host(gn.col), host(gn.val))
    a = go.val.astype(np.float64)
    x = features(cfg.n, cfg.f, cfg.ld, seed=2)
    p = GCNParams.init(cfg.f, 128, 41, DEV, seed=1)
    h1 = host(G.gsp_gcn_layer(gn, dev(x), p.w1, p.b1, "relu"))
    out = host(gcn_inference(gn, dev(x), p))
    rng = np.random.default_rng(0)
    rows = rng.choice(cfg.n, 60, replace=False)
    x602 = np.ascontiguousarray(x[:, :cfg.f])
    w1, b1, w2, b2 = host(p.w1), host(p.b1), host(p.w2), host(p.b2)
    for r in rows:
        yr, c = orc.gcn_layer(go.row_ptr, go.col, a, x602, w1, b1, "relu", r0=r, r1=r + 1)
        assert_within(h1[r:r + 1], yr, c, rel=_lin_rel(cfg.f), what=f"layer1 row {r}")
        y2, c2 = orc.gcn_layer(go.row_ptr, go.col, a, h1, w2, b2, "none", r0=r, r1=r + 1)
        assert_within(out[r:r + 1], y2, c2, rel=_lin_rel(128), what=f"layer2 row {r}")


@pytest.mark.parametrize("hidden", [128, 512], ids=["4x32", "4x128"])
def test_gat_inference_end_to_end_small(built, hidden):
    """2-layer GAT through inference.gat_inference vs the oracle composed from
    the GPU's own layer-1 intermediates (linear, attention projection, fused
    aggregate with ELU; output layer with one 41-wide head).  Both readings of
    A20 ("hidden size 128 ... 4 attention heads"): 4 x 32 and 4 x 128."""
    from paper_2103_00959_b200.inference import GATParams, gat_inference, _padded
    go, gg, _, _ = built["cl4000"]
    n = go.n
    d1 = hidden // 4
    x = uniform((n, 50), seed=1)
    p = GATParams.init(50, hidden, 4, 41, DEV, seed=2)
    out = host(gat_inference(gg, dev(x), p))
    z1 = G.gsp_linear(dev(x), p.w1, y=_padded(n, hidden, DEV))
    el1, er1 = G.gsp_attn_project(z1, p.al1, p.ar1, 4, d1)
    # layer 1 against the oracle on the GPU's own z1, el1, er1
    s1 = orc.gat_scores(go.row_ptr, go.col, host(el1), host(er1), 4)
    a1 = orc.edge_softmax(go.row_ptr, s1, 4)
    y1r, c1 = orc.multihead_spmm(go.row_ptr, go.col, a1, host(z1), 4, d1)
    h1 = G.gsp_gat_aggregate_bias_act(gg, el1, er1, z1, 4, d1, p.b1, "elu", y=_padded(n, hidden, DEV))
    assert_within(host(h1), orc.bias_act(y1r, host(p.b1), "elu"), c1, what=f"gat layer 1 ({hidden})")
    z2 = G.gsp_linear(h1, p.w2, y=_padded(n, 41, DEV))
    el2, er2 = G.gsp_attn_project(z2, p.al2, p.ar2, 1, 41)
    s = orc.gat_scores(go.row_ptr, go.col, host(el2), host(er2), 1)
    al = orc.edge_softmax(go.row_ptr, s, 1)
    yr, c = orc.multihead_spmm(go.row_ptr, go.col, al, host(z2), 1, 41)
    assert_within(out, orc.bias_act(yr, host(p.b2), "none"), c, what="gat output layer")


# ---------------------------------------------------------------- single head, padded rows

def _padded_view(a, ld):
    t = torch.zeros((a.shape[0], ld), dtype=torch.float32, device=DEV)
    t[:, :a.shape[1]] = dev(a)
    return t[:, :a.shape[1]]


@pytest.mark.parametrize("D", [1, 2, 3])
def test_single_head_padded_z(built, D):
    """H = 1 with d < 4 and ldz = 4: the plain plan's slab is wider than d, so a
    team must still hold ONE head (engine_hpt caps at the head count).  Covers
    multi-head SpMM, both GAT schedules and the aggregate backward."""
    H = 1
    for name in ("multi0", "cl4000", "hubs"):
        go, gg, _, _ = built[name]
        n = go.n
        z = uniform((n, H * D), seed=3)
        zt = _padded_view(z, 4)
        alpha = uniform((go.nnz, H), seed=4, low=0, high=1)
        yref, cond = orc.multihead_spmm(go.row_ptr, go.col, alpha.astype(np.float64), z, H, D)
        assert_within(host(G.gsp_multihead_spmm(gg, dev(alpha), zt, H, D)), yref, cond, what=f"mh {name} D={D}")
        el = uniform((n, H), seed=4, low=-3, high=3)
        er = uniform((n, H), seed=5, low=-3, high=3)
        yref, cond, aref = _gat_ref(go, el, er, z, H, D, 0.2)
        for single in (False, True):
            y, a = G.gsp_gat_aggregate(gg, dev(el), dev(er), zt, H, D, 0.2, alpha_out=True, single_launch=single)
            assert_within(host(y), yref, cond, what=f"gat {name} D={D} single={single}")
            assert np.all(np.abs(host(a) - aref) <= 1e-5 * aref + 1e-9), (name, D, single)
        dy = uniform((n, H * D), seed=7)
        at, perm = G.gsp_csr_transpose(gg)
        dz, d_el, d_er = [host(t) for t in G.gsp_gat_aggregate_backward(gg, at, perm, dev(el), dev(er), zt,
                                                                         _padded_view(dy, 4), H, D)]
        dz_r, del_r, der_r, _ = orc.gat_backward(go.row_ptr, go.col, el, er, z, dy, H, D)
        rp_t, ct, pm = orc.csr_transpose(go.row_ptr, go.col, n)
        dz_c, _ = orc.multihead_spmm(rp_t, ct, aref[pm], np.abs(dy), H, D)
        assert_within(dz, dz_r, dz_c, what=f"dz {name} D={D}")


@pytest.mark.parametrize("classes", [1, 2])
def test_gat_inference_few_classes(built, classes):
    """gat_inference's output layer is one head of `classes` columns in a padded
    buffer (ld 4): the case that used to form hpt > 1 for a single head."""
    from paper_2103_00959_b200.inference import GATParams, gat_inference, _padded
    go, gg, _, _ = built["cl4000"]
    n = go.n
    x = uniform((n, 50), seed=1)
    p = GATParams.init(50, 64, 4, classes, DEV, seed=2)
    out = host(gat_inference(gg, dev(x), p))
    z1 = G.gsp_linear(dev(x), p.w1, y=_padded(n, 64, DEV))
    el1, er1 = G.gsp_attn_project(z1, p.al1, p.ar1, 4, 16)
    h1 = G.gsp_gat_aggregate_bias_act(gg, el1, er1, z1, 4, 16, p.b1, "elu", y=_padded(n, 64, DEV))
    z2 = G.gsp_linear(h1, p.w2, y=_padded(n, classes, DEV))
    el2, er2 = G.gsp_attn_project(z2, p.al2, p.ar2, 1, classes)
    s = orc.gat_scores(go.row_ptr, go.col, host(el2), host(er2), 1)
    al = orc.edge_softmax(go.row_ptr, s, 1)
    yr, c = orc.multihead_spmm(go.row_ptr, go.col, al, host(z2), 1, classes)
    assert_within(out, orc.bias_act(yr, host(p.b2), "none"), c, what=f"gat output layer classes={classes}")


# ---------------------------------------------------------------- GSP_VALIDATE, nullable deg_out

def test_validate_mode_rejects_nonfinite(built):
    go, gg, _, _ = built["cl4000"]
    H, D = 2, 8
    n = go.n
    z = dev(uniform((n, H * D), seed=3))
    el = dev(uniform((n, H), seed=4, low=-3, high=3))
    er = dev(uniform((n, H), seed=5, low=-3, high=3))
    lg = dev(uniform((go.nnz, H), seed=6))
    y0 = G.gsp_gat_aggregate(gg, el, er, z, H, D)
    G.gsp_set_flags(G.GSP_VALIDATE)
    try:
        assert torch.equal(G.gsp_gat_aggregate(gg, el, er, z, H, D), y0)  # finite input: same result
        a0 = G.gsp_edge_softmax(gg, lg, H)
        for bad in (float("nan"), float("inf"), -float("inf")):
            er2 = er.clone()
            er2[n // 2, 1] = bad
            y = torch.full((n, H * D), 7.0, device=DEV)
            with pytest.raises(G.GspError) as e:
                G.gsp_gat_aggregate(gg, el, er2, z, H, D, y=y)
            assert e.value.status == 4 and "er" in str(e.value)
            assert torch.all(y == 7.0)  # outputs untouched
            lg2 = lg.clone()
            lg2[go.nnz - 1, 0] = bad
            with pytest.raises(G.GspError) as e:
                G.gsp_edge_softmax(gg, lg2, H)
            assert e.value.status == 4
        el2 = el.clone()
        el2[0, 0] = float("nan")
        at, perm = G.gsp_csr_transpose(gg)
        with pytest.raises(G.GspError):
            G.gsp_gat_aggregate_backward(gg, at, perm, el2, er, z, z, H, D)
        assert torch.equal(G.gsp_edge_softmax(gg, lg, H), a0)
    finally:
        G.gsp_set_flags(0)
    # outside validate mode a NaN stays inside its row (A12)
    lg2 = lg.clone()
    r = 17
    lg2[int(go.row_ptr[r]), 0] = float("nan")
    a = host(G.gsp_edge_softmax(gg, lg2, H))
    rows = np.repeat(np.arange(n), np.diff(go.row_ptr))
    assert np.all(np.isnan(a[rows == r, 0])) and np.all(np.isfinite(a[rows != r]))


def test_normalize_without_deg_out(built):
    for name in ("isolated-nofill", "multi1", "cl4000", "star100k"):
        go, gg, (deg, a64, a32), gn = built[name]
        g2 = G.gsp_sym_normalize(gg, keep_deg=False)
        assert g2.deg is None
        np.testing.assert_array_equal(host(g2.val).view(np.uint32), a32.view(np.uint32), err_msg=name)
