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
