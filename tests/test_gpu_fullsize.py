"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (default gsp_spmm plan): the CSR is compared bit-exactly, the outputs on
sampled rows (random + the heaviest hub rows) against the oracle computed row
by row, and properties that hold at any size on every row."""
import numpy as np
import pytest
import torch

import oracle as orc
import paper_2103_00959_b200 as G
from synth import CONFIGS, features, graph_for, uniform
from test_gpu_parity import DEV, assert_within, dev, host

pytestmark = pytest.mark.gpu


def _sample_rows(row_ptr, k=400, seed=0):
    deg = np.diff(row_ptr)
    rng = np.random.default_rng(seed)
    rows = set(rng.choice(deg.size, size=min(k, deg.size), replace=False).tolist())
    rows |= set(np.argsort(deg)[-16:].tolist())
    return sorted(rows)


@pytest.fixture(scope="module")
def c4():
    cfg = CONFIGS["C4"]
    s, d = graph_for(cfg, seed=1)
    go = orc.build_csr(cfg.n, s, d, None, True, 1.0)
    deg, a64, a32 = orc.sym_norm(go)
    gg = G.gsp_coo_to_csr(cfg.n, dev(s), dev(d), None, True, 1.0)
    gn = G.gsp_sym_normalize(gg)
    return cfg, go, (deg, a64, a32), gg, gn


def test_c4_csr_bit_exact(c4):
    cfg, go, (deg, a64, a32), gg, gn = c4
    assert gg.nnz == go.nnz == cfg.nnz
    np.testing.assert_array_equal(host(gg.row_ptr), go.row_ptr)
    np.testing.assert_array_equal(host(gg.col), go.col)
    np.testing.assert_array_equal(host(gg.val), go.val)
    np.testing.assert_array_equal(host(gn.deg), deg)
    np.testing.assert_array_equal(host(gn.val).view(np.uint32), a32.view(np.uint32))


def test_c4_spmm_sampled_rows(c4):
    cfg, go, (deg, a64, a32), gg, gn = c4
    x = features(cfg.n, cfg.f, cfg.ld, seed=2)
    xt = dev(x)
    y = host(G.gsp_spmm(gn, xt, f=cfg.f))
    for r in _sample_rows(go.row_ptr):
        yr, cr = orc.spmm(go.row_ptr, go.col, a64, x, f=cfg.f, r0=r, r1=r + 1)
        assert_within(y[r:r + 1], yr, cr, what=f"C4 row {r} (deg {go.row_ptr[r + 1] - go.row_ptr[r]})")
    # determinism at full size
    y2 = host(G.gsp_spmm(gn, xt, f=cfg.f))
    assert np.array_equal(y, y2)


def test_c4_spmm_blocked_sampled_rows(c4):
    """The column-blocked SpMM in bench.py's headline plan (G.colblock_bounds:
    two column halves on C4) at full size: sampled rows + the 16 heaviest
    hubs vs the oracle, the identity A^ sqrt(d) = sqrt(d) on every row, and
    determinism."""
    cfg, go, (deg, a64, a32), gg, gn = c4
    bounds = G.colblock_bounds(gn, cfg.f)
    assert len(bounds) == 3, bounds
    blocks = G.gsp_csr_colblock(gn, bounds)
    assert sum(blocks.nnz) == gn.nnz
    x = G.empty_features(cfg.n, cfg.f, torch.device(DEV))
    xh = features(cfg.n, cfg.f, cfg.f, seed=2)
    x.copy_(dev(xh))
    y = host(G.gsp_spmm_blocked(blocks, x, f=cfg.f))
    for r in _sample_rows(go.row_ptr):
        yr, cr = orc.spmm(go.row_ptr, go.col, a64, xh, f=cfg.f, r0=r, r1=r + 1)
        assert_within(y[r:r + 1, :cfg.f], yr, cr, what=f"C4 blocked row {r}")
    assert np.array_equal(y, host(G.gsp_spmm_blocked(blocks, x, f=cfg.f)))
    s8 = torch.sqrt(gn.deg).float()[:, None].repeat(1, 8).contiguous()
    np.testing.assert_allclose(host(G.gsp_spmm_blocked(blocks, s8)), np.sqrt(deg)[:, None].repeat(8, 1), rtol=3e-6)


def test_c4_spmm_f16_sampled_rows(c4):
    """gsp_spmm_f16 at full size (bench's C4_spmm_f16_storage line) vs the oracle
    on the fp16 values, sampled rows incl. the heaviest hubs."""
    cfg, go, (deg, a64, a32), gg, gn = c4
    x = features(cfg.n, cfg.f, cfg.ld, seed=2)
    xh = x.astype(np.float16)
    y = host(G.gsp_spmm_f16(gn, torch.from_numpy(xh).to(DEV), f=cfg.f))
    x64 = xh.astype(np.float64)
    for r in _sample_rows(go.row_ptr, k=200, seed=1):
        yr, cr = orc.spmm(go.row_ptr, go.col, a64, x64, f=cfg.f, r0=r, r1=r + 1)
        assert_within(y[r:r + 1], yr, cr, what=f"C4 f16 row {r}")


def test_c4_linear_tensor_cores_sampled_rows():
    """The NEXT-1 layer-1 GEMM shape (232,965 x 602 -> 128) on the tcgen05 path
    vs the oracle's dense product on sampled rows (3xTF32 bound)."""
    from test_gpu_parity import _tc_rel
    cfg = CONFIGS["C4"]
    x = features(cfg.n, cfg.f, cfg.ld, seed=2)
    w = uniform((cfg.f, 128), seed=7)
    y = host(G.gsp_linear(dev(x)[:, :cfg.f], dev(w)))
    rows = np.random.default_rng(3).choice(cfg.n, 300, replace=False)
    rows = np.concatenate([rows, [0, cfg.n - 1]])
    yr, c = orc.linear(x[rows, :cfg.f].copy(), w)
    assert_within(y[rows], yr, c, rel=_tc_rel(cfg.f), what="C4 layer-1 GEMM")


def test_c4_identity_every_row(c4):
    """I1: A^ sqrt(d) = sqrt(d) on all 232,965 rows."""
    cfg, go, (deg, a64, a32), gg, gn = c4
    x = torch.sqrt(gn.deg).float()[:, None].repeat(1, 8).contiguous()
    y = host(G.gsp_spmm(gn, x))
    np.testing.assert_allclose(y, np.sqrt(deg)[:, None].repeat(8, 1), rtol=3e-6)


def test_c4_propagate_eigenvector(c4):
    """A^ sqrt(d) = sqrt(d) => K=10 PPR propagation of sqrt(d) is (sum theta) sqrt(d) on every row."""
    cfg, go, (deg, a64, a32), gg, gn = c4
    th = orc.ppr_coeffs(0.1, 10)
    x = torch.sqrt(gn.deg).float()[:, None].repeat(1, 4).contiguous()
    y = host(G.gsp_propagate(gn, x, th))
    np.testing.assert_allclose(y, th.sum() * np.sqrt(deg)[:, None].repeat(4, 1), rtol=3e-5)


def test_c3_gat_sampled_rows_and_convexity():
    cfg = CONFIGS["C3"]
    H, D = cfg.heads, cfg.d
    s, d = graph_for(cfg, seed=1)
    go = orc.build_csr(cfg.n, s, d, None, True, 1.0)
    gg = G.gsp_coo_to_csr(cfg.n, dev(s), dev(d), None, True, 1.0)
    np.testing.assert_array_equal(host(gg.col), go.col)
    z = uniform((cfg.n, H * D), seed=3)
    al = uniform((H, D), seed=6)
    ar = uniform((H, D), seed=7)
    zt = dev(z)
    el, er = G.gsp_attn_project(zt, dev(al.reshape(-1)), dev(ar.reshape(-1)), H, D)
    rows = _sample_rows(go.row_ptr, k=200)
    el_ref, er_ref, elc, erc = orc.attn_project(z, al, ar, H, D)
    assert_within(host(el), el_ref, elc, what="el")
    assert_within(host(er), er_ref, erc, what="er")
    y, alpha = G.gsp_gat_aggregate(gg, el, er, zt, H, D, 0.2, alpha_out=True)
    y = host(y)
    sc = orc.gat_scores(go.row_ptr, go.col, host(el), host(er), H, 0.2)
    aref = orc.edge_softmax(go.row_ptr, sc, H)
    err = np.abs(host(alpha) - aref)
    assert np.all(err <= 1e-5 * aref + 1e-9)
    for r in rows:
        yr, cr = orc.multihead_spmm(go.row_ptr, go.col, aref, z, H, D, r0=r, r1=r + 1)
        assert_within(y[r:r + 1], yr, cr, what=f"C3 row {r}")
    # convexity at full size: constant per-head features are reproduced
    zc = torch.arange(1, H + 1, device=DEV, dtype=torch.float32).repeat_interleave(D)[None, :].repeat(cfg.n, 1)
    yc = G.gsp_gat_aggregate(gg, el, er, zc.contiguous(), H, D, 0.2)
    torch.testing.assert_close(yc, zc, rtol=2e-6, atol=0)


# ---------------------------------------------------------------- C1, C2, C2g: full output
def _built(key, seed=1):
    cfg = CONFIGS[key]
    s, d = graph_for(cfg, seed=seed)
    go = orc.build_csr(cfg.n, s, d, None, True, 1.0)
    no = orc.sym_norm(go)
    gg = G.gsp_coo_to_csr(cfg.n, dev(s), dev(d), None, True, 1.0)
    gn = G.gsp_sym_normalize(gg)
    return cfg, go, no, gg, gn


def _csr_bit_exact(cfg, go, no, gg, gn):
    deg, a64, a32 = no
    assert gg.nnz == go.nnz
    np.testing.assert_array_equal(host(gg.row_ptr), go.row_ptr)
    np.testing.assert_array_equal(host(gg.col), go.col)
    np.testing.assert_array_equal(host(gg.val).view(np.uint32), go.val.view(np.uint32))
    np.testing.assert_array_equal(host(gn.deg), deg)
    np.testing.assert_array_equal(host(gn.val).view(np.uint32), a32.view(np.uint32))


@pytest.mark.parametrize("key", ["C1", "C2"])
def test_small_configs_full_output(key):
    """C1 (Cora-shaped, F = 1433) and C2 (Pubmed-shaped, F = 500) at their exact
    shapes: CSR and A^ bit-exact, every output element within the bound, for
    dense U[-1,1) features and binary bag-of-words features."""
    cfg, go, no, gg, gn = _built(key)
    _csr_bit_exact(cfg, go, no, gg, gn)
    deg, a64, a32 = no
    assert go.nnz == cfg.nnz
    for x in (features(cfg.n, cfg.f, cfg.ld, seed=2), bag_of_words_ld(cfg)):
        y = host(G.gsp_spmm(gn, dev(x), f=cfg.f))
        yref, cond = orc.spmm(go.row_ptr, go.col, a64, x, f=cfg.f)
        assert_within(y, yref, cond, what=f"{cfg.name} full output")


def bag_of_words_ld(cfg):
    from synth import bag_of_words
    x = np.zeros((cfg.n, cfg.ld), np.float32)
    x[:, :cfg.f] = bag_of_words(cfg.n, cfg.f, seed=3)
    return x


@pytest.mark.parametrize("H,D", [(8, 8), (8, 64)])
def test_c2g_gat_full_output(H, D):
    """C2g (Pubmed-shaped GAT, 8 heads x 8 = the standard hidden layer, and 8 x
    64): attention projection, every alpha and every output element, both
    schedules of gsp_gat_aggregate, and the standalone a6 / a7 calls."""
    cfg, go, no, gg, gn = _built("C2g")
    n = cfg.n
    z = uniform((n, H * D), seed=3)
    al, ar = uniform((H, D), seed=6), uniform((H, D), seed=7)
    el, er = G.gsp_attn_project(dev(z), dev(al.reshape(-1)), dev(ar.reshape(-1)), H, D)
    el_ref, er_ref, elc, erc = orc.attn_project(z, al, ar, H, D)
    assert_within(host(el), el_ref, elc, what="el")
    assert_within(host(er), er_ref, erc, what="er")
    sc = orc.gat_scores(go.row_ptr, go.col, host(el), host(er), H, 0.2)
    aref = orc.edge_softmax(go.row_ptr, sc, H)
    yref, cond = orc.multihead_spmm(go.row_ptr, go.col, aref, z, H, D)
    for single in (False, True):
        y, a = G.gsp_gat_aggregate(gg, el, er, dev(z), H, D, 0.2, alpha_out=True, single_launch=single)
        assert_within(host(y), yref, cond, what=f"C2g {H}x{D} single={single}")
        assert np.all(np.abs(host(a) - aref) <= 1e-5 * aref + 1e-9)
    # standalone a6 on the oracle's own scores (as fp32 logits) and a7 on the oracle's alpha
    lg = sc.astype(np.float32)
    a6 = host(G.gsp_edge_softmax(gg, dev(lg), H))
    a6ref = orc.edge_softmax(go.row_ptr, lg.astype(np.float64), H)
    assert np.all(np.abs(a6 - a6ref) <= 1e-5 * a6ref + 1e-9)
    a32 = aref.astype(np.float32)
    y7 = host(G.gsp_multihead_spmm(gg, dev(a32), dev(z), H, D))
    y7ref, c7 = orc.multihead_spmm(go.row_ptr, go.col, a32.astype(np.float64), z, H, D)
    assert_within(y7, y7ref, c7, what=f"C2g a7 {H}x{D}")


# ---------------------------------------------------------------- C5: the 2 x 128 + 64 plan at full size
def test_c5_full_size():
    """C5 (Yelp-shaped, F = 300): CSR bit-exact; bench's launch plan (two
    128-column slabs + a 64-column tail launch); sampled rows and the 16
    heaviest hubs vs the oracle; A^ sqrt(d) = sqrt(d) on every row."""
    cfg, go, no, gg, gn = _built("C5")
    _csr_bit_exact(cfg, go, no, gg, gn)
    deg, a64, a32 = no
    x = features(cfg.n, cfg.f, cfg.ld, seed=2)
    xt = dev(x)
    assert G.gsp_spmm_plan_info(gn, xt, cfg.f) == (2, 128, 64)
    y = host(G.gsp_spmm(gn, xt, f=cfg.f))
    for r in _sample_rows(go.row_ptr, k=400, seed=5):
        yr, cr = orc.spmm(go.row_ptr, go.col, a64, x, f=cfg.f, r0=r, r1=r + 1)
        assert_within(y[r:r + 1], yr, cr, what=f"C5 row {r} (deg {go.row_ptr[r + 1] - go.row_ptr[r]})")
    del xt
    xs = torch.sqrt(gn.deg).float()[:, None].repeat(1, 8).contiguous()
    np.testing.assert_allclose(host(G.gsp_spmm(gn, xs)), np.sqrt(deg)[:, None].repeat(8, 1), rtol=3e-6)


def _emulated_partition_bitwise(gn, x, f, P):
    """The P-rank row partition on one GPU: per-rank slices over the padded
    all-gather layout give rows bitwise equal to the single-GPU SpMM (§8(e))."""
    y_global = G.gsp_spmm(gn, x, f=f)
    b, _ = G.gsp_partition_rows(gn, P)
    npad = int(np.diff(b).max())
    xg = torch.zeros((P * npad, x.shape[1]), dtype=torch.float32, device=DEV)
    for q in range(P):
        xg[q * npad:q * npad + b[q + 1] - b[q]] = x[b[q]:b[q + 1]]
    for r in range(P):
        sl = G.gsp_csr_slice(gn, b, r, npad)
        yl = G.gsp_spmm(sl, xg, f=f)
        assert torch.equal(yl, y_global[b[r]:b[r + 1]]), f"rank {r} of {P}"
    return b


def test_c4_partition_p8_bitwise(c4):
    """C4 at P = 8 (the scaling configuration), emulated on one GPU."""
    cfg, go, (deg, a64, a32), gg, gn = c4
    x = dev(features(cfg.n, cfg.f, cfg.ld, seed=2))
    b = _emulated_partition_bitwise(gn, x, cfg.f, 8)
    np.testing.assert_array_equal(np.array(b), orc.partition_rows(go.row_ptr, 8))


# ---------------------------------------------------------------- C6: Yelp x10, streamed
@pytest.fixture(scope="module")
def c6():
    return _built("C6")


def test_c6_csr_bit_exact(c6):
    cfg, go, no, gg, gn = c6
    assert go.nnz == cfg.nnz == gg.nnz
    _csr_bit_exact(cfg, go, no, gg, gn)


def test_c6_spmm_streamed_rows_identity_and_partition(c6):
    """C6 (7.17M nodes, 147M nnz, X = 8.6 GB): sampled rows + the 16 heaviest
    hubs through the oracle's row-range entry point; A^ sqrt(d) = sqrt(d) on
    every row; the P = 8 row partition (emulated) bitwise equal on every row."""
    cfg, go, no, gg, gn = c6
    deg, a64, a32 = no
    x = features(cfg.n, cfg.f, cfg.ld, seed=2)
    xt = dev(x)
    y = G.gsp_spmm(gn, xt, f=cfg.f)
    rows = _sample_rows(go.row_ptr, k=300, seed=6)
    yh = host(y[torch.tensor(rows, device=DEV)])
    for i, r in enumerate(rows):
        yr, cr = orc.spmm(go.row_ptr, go.col, a64, x, f=cfg.f, r0=r, r1=r + 1)
        assert_within(yh[i:i + 1], yr, cr, what=f"C6 row {r} (deg {go.row_ptr[r + 1] - go.row_ptr[r]})")
    del y
    b = _emulated_partition_bitwise(gn, xt, cfg.f, 8)
    np.testing.assert_array_equal(np.array(b), orc.partition_rows(go.row_ptr, 8))
    del xt
    xs = torch.sqrt(gn.deg).float()[:, None].repeat(1, 4).contiguous()
    np.testing.assert_allclose(host(G.gsp_spmm(gn, xs)), np.sqrt(deg)[:, None].repeat(4, 1), rtol=3e-6)
