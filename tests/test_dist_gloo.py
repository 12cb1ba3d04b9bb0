"""Multi-process (world size 2 and 3, gloo, CPU) tests of the row-partitioned
SpMM driver paper_2103_00959_b200.dist.RowPartitionedSpMM: partition, padded
all-gather layout, feature chunking and shard assembly.  The per-rank compute
steps are the oracle's (injected as `ops`), so these run without a GPU; the
CUDA kernels behind the same steps are checked on one GPU by
test_gpu_parity.py::test_partition_slice_bit_exact_and_invariant."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as orc
from synth import chung_lu, features


class OracleCSR:
    def __init__(self, row_ptr, col, val, n_cols):
        self.row_ptr, self.col, self.val, self.n_cols = row_ptr, col, val, n_cols
        self.n_rows = row_ptr.size - 1


class OracleOps:
    """Host stand-ins for gsp_partition_rows / gsp_csr_slice / gsp_spmm."""

    @staticmethod
    def partition(a, parts):
        return orc.partition_rows(a.row_ptr, parts)

    @staticmethod
    def slice(a, bounds, rank, npad):
        rp, co, vo = orc.csr_slice(a.row_ptr, a.col, a.val, np.asarray(bounds), rank, npad)
        return OracleCSR(rp, co, vo, len(bounds) * npad - npad)

    @staticmethod
    def spmm(local, x, f, y):
        yy, _ = orc.spmm(local.row_ptr, local.col, local.val.astype(np.float64), x.numpy(), f=f, want_cond=False)
        y.copy_(torch.from_numpy(yy.astype(np.float32)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gather(out, inp):
    parts = list(out.chunk(dist.get_world_size(), dim=0))
    dist.all_gather(parts, inp.contiguous())
    out.copy_(torch.cat(parts, 0))


def _worker(rank, world, port, n, m, f, chunks, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2103_00959_b200.dist import RowPartitionedSpMM
        s, d = chung_lu(n, m, seed=3)
        g = orc.build_csr(n, s, d, None, True, 1.0)
        _, _, a32 = orc.sym_norm(g)
        a = OracleCSR(g.row_ptr, g.col, a32, n)
        x = features(n, f, seed=4)
        op = RowPartitionedSpMM(a, rank, world, f, chunks=chunks, all_gather=_gather, device="cpu", ops=OracleOps)
        op.load_shard(torch.from_numpy(x[op.r0:op.r1]))
        y = op()
        yref, _ = orc.spmm(g.row_ptr, g.col, a32.astype(np.float64), x, want_cond=False)
        ok = np.array_equal(y.numpy(), yref[op.r0:op.r1].astype(np.float32))
        q.put((rank, ok, op.r0, op.r1, op.npad, op.cols))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,chunks", [(2, 1), (2, 3), (3, 4)])
def test_row_partitioned_spmm_gloo(world, chunks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n, m, f = 3000, 20000, 300
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, m, f, chunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(ok for _, ok, *_ in res), res
    # the row blocks tile [0, n) and the chunks tile [0, f)
    assert res[0][2] == 0 and res[-1][3] == n
    for a, b in zip(res[:-1], res[1:]):
        assert a[3] == b[2]
    cols = res[0][5]
    assert cols[0] == 0 and cols[-1] == f and all(c % 128 == 0 for c in cols[:-1])


def test_chunk_bounds_and_padding():
    from paper_2103_00959_b200.dist import chunk_bounds, padded_rows
    assert chunk_bounds(602, 4, align=4) == [0, 152, 304, 456, 602]
    assert chunk_bounds(602, 5) == [0, 128, 256, 384, 512, 602]
    assert chunk_bounds(602, 4) == [0, 256, 512, 602]
    assert chunk_bounds(3, 4) == [0, 3]
    assert chunk_bounds(8, 1) == [0, 8]
    assert padded_rows([0, 5, 5, 12]) == 7


class OracleGatOps(OracleOps):
    """Host stand-ins for gsp_attn_project / gsp_gat_aggregate (fp64 oracle,
    rounded to fp32 where the product's outputs are fp32)."""

    @staticmethod
    def attn_project(z, a_l, a_r, heads, d, el, er):
        e_l, e_r, _, _ = orc.attn_project(z.numpy(), a_l.numpy().reshape(heads, d), a_r.numpy().reshape(heads, d),
                                          heads, d)
        el.copy_(torch.from_numpy(e_l.astype(np.float32)))
        er.copy_(torch.from_numpy(e_r.astype(np.float32)))

    @staticmethod
    def gat_aggregate(local, el, er, z, heads, d, slope, y, ws):
        sc = orc.gat_scores(local.row_ptr, local.col, el.numpy(), er.numpy(), heads, slope)
        al = orc.edge_softmax(local.row_ptr, sc, heads)
        yy, _ = orc.multihead_spmm(local.row_ptr, local.col, al, z.numpy(), heads, d, want_cond=False)
        y.copy_(torch.from_numpy(yy.astype(np.float32)))


def _gat_worker(rank, world, port, n, m, H, D, groups, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2103_00959_b200.dist import RowPartitionedGAT
        from synth import uniform
        s, d = chung_lu(n, m, seed=5)
        g = orc.build_csr(n, s, d, None, True, 1.0)
        a = OracleCSR(g.row_ptr, g.col, g.val, n)
        z = uniform((n, H * D), seed=3)
        al, ar = uniform(H * D, seed=6), uniform(H * D, seed=7)
        op = RowPartitionedGAT(a, rank, world, H, D, head_groups=groups, all_gather=_gather, device="cpu",
                               ops=OracleGatOps)
        op.load_shard(torch.from_numpy(z[op.r0:op.r1]))
        y = op(torch.from_numpy(al), torch.from_numpy(ar)).numpy()
        # global reference: the same oracle steps on the whole graph
        el, er, _, _ = orc.attn_project(z, al.reshape(H, D), ar.reshape(H, D), H, D)
        yref = np.zeros((n, H * D), np.float32)
        for h0, h1 in zip(op.hg[:-1], op.hg[1:]):
            hc = h1 - h0
            sc = orc.gat_scores(g.row_ptr, g.col, el[:, h0:h1].astype(np.float32).copy(),
                                er[:, h0:h1].astype(np.float32).copy(), hc, 0.2)
            yy, _ = orc.multihead_spmm(g.row_ptr, g.col, orc.edge_softmax(g.row_ptr, sc, hc),
                                       np.ascontiguousarray(z[:, h0 * D:h1 * D]), hc, D, want_cond=False)
            yref[:, h0 * D:h1 * D] = yy
        q.put((rank, bool(np.array_equal(y, yref[op.r0:op.r1])), op.r0, op.r1, op.hg))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,groups", [(2, 1), (2, 4), (3, 2)])
def test_row_partitioned_gat_gloo(world, groups):
    """RowPartitionedGAT (all-gather Z and er, el local) over gloo
    with the oracle's per-rank steps equals the global oracle exactly."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n, m, H, D = 2500, 15000, 8, 32
    procs = [ctx.Process(target=_gat_worker, args=(r, world, port, n, m, H, D, groups, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, *_ in res), res
    assert res[0][2] == 0 and res[-1][3] == n
    hg = res[0][4]
    from paper_2103_00959_b200.dist import head_chunks
    assert hg == head_chunks(H, D, groups) and (groups == 1) == (len(hg) == 2)


def test_head_chunks():
    from paper_2103_00959_b200.dist import head_chunks
    assert head_chunks(8, 64, 1) == [0, 8]
    assert head_chunks(8, 64, 4) == [0, 2, 4, 6, 8]   # 128-column groups
    assert head_chunks(8, 64, 8) == [0, 2, 4, 6, 8]   # never narrower than one slab when avoidable
    assert head_chunks(4, 128, 4) == [0, 1, 2, 3, 4]
    assert head_chunks(3, 16, 2) == [0, 2, 3]


def test_remap_col_bounds_keeps_block_membership():
    """Column blocks under the row partition: a column's block in the gathered
    layout (gsp_csr_slice's remap q * npad + c - b_q) is its global block."""
    from paper_2103_00959_b200.dist import padded_rows, remap_col_bounds
    rng = np.random.default_rng(3)
    for _ in range(50):
        n = int(rng.integers(5, 400))
        world = int(rng.integers(1, 6))
        cuts = sorted(rng.integers(0, n + 1, world - 1).tolist())
        bounds = [0] + cuts + [n]
        npad = max(1, padded_rows(bounds))
        kb = int(rng.integers(1, 5))
        cb = [0] + sorted(rng.integers(0, n + 1, kb - 1).tolist()) + [n]
        rb = remap_col_bounds(cb, bounds, npad)
        assert rb[0] == 0 and rb[-1] == world * npad and rb == sorted(rb)
        for c in range(n):
            q = max(p for p in range(world) if bounds[p] <= c < bounds[p + 1])
            r = q * npad + c - bounds[q]
            kg = max(k for k in range(kb) if cb[k] <= c)
            kr = max(k for k in range(kb) if rb[k] <= r)
            assert kg == kr, (n, bounds, cb, c)
