"""The multi-GPU product path (RowPartitionedSpMM with the libgsp kernels) on
the one GPU a test box has: P ranks share cuda:0 and exchange their padded X
shards through a gloo all-gather staged via host memory (NCCL refuses two ranks
on one device), plus a world-size-1 NCCL run of the same driver.  Each rank's Y
shard must be bitwise equal to the single-process gsp_spmm result (DESIGN.md
§6, §9)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _staged_gather(out, inp):
    parts = [torch.empty_like(inp, device="cpu") for _ in range(dist.get_world_size())]
    dist.all_gather(parts, inp.cpu())
    out.copy_(torch.cat(parts, 0))


def _worker(rank, world, port, backend, chunks, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2103_00959_b200 as G
        from paper_2103_00959_b200.dist import RowPartitionedSpMM
        from synth import chung_lu, features
        n, m, f = 20000, 150000, 300
        s, d = chung_lu(n, m, seed=5)
        dev = torch.device("cuda", 0)
        g = G.gsp_sym_normalize(G.gsp_coo_to_csr(n, torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev)))
        x = torch.from_numpy(features(n, f, (f + 3) // 4 * 4, seed=6)).to(dev)
        y_ref = G.gsp_spmm(g, x, f=f)
        op = RowPartitionedSpMM(g, rank, world, f, chunks=chunks, device=dev,
                                all_gather=None if backend == "nccl" else _staged_gather)
        op.load_shard(x[op.r0:op.r1, :f])
        y = op()
        torch.cuda.synchronize()
        ok = torch.equal(y, y_ref[op.r0:op.r1])
        # column blocks: global bounds mapped into each slice's gathered layout
        # give the single-GPU gsp_spmm_blocked bitwise
        cb = [0, n // 3, 2 * n // 3, n]
        ob = RowPartitionedSpMM(g, rank, world, f, chunks=chunks, device=dev, col_blocks=cb,
                                all_gather=None if backend == "nccl" else _staged_gather)
        ob.load_shard(x[ob.r0:ob.r1, :f])
        yb = ob()
        torch.cuda.synchronize()
        ok = ok and torch.equal(yb, G.gsp_spmm_blocked(G.gsp_csr_colblock(g, cb), x, f=f)[ob.r0:ob.r1])
        # K-step propagation through the same partition (NEXT-4)
        from paper_2103_00959_b200.dist import RowPartitionedPropagate
        th = [0.1 * 0.9 ** k for k in range(6)]
        pp = RowPartitionedPropagate(g, rank, world, f, chunks=chunks, device=dev,
                                     all_gather=None if backend == "nccl" else _staged_gather)
        pp.load_shard(x[pp.r0:pp.r1, :f])
        yp = pp(th)
        torch.cuda.synchronize()
        ok = ok and torch.equal(yp, G.gsp_propagate(g, x, th, f=f)[pp.r0:pp.r1])
        # GAT (all-gather Z and er, el local); head_groups = 1 is
        # bitwise equal to the single-GPU attn_project + gat_aggregate, more
        # groups to the single-GPU calls on the same head groups
        from paper_2103_00959_b200.dist import RowPartitionedGAT
        from synth import uniform
        H, D = 8, 32
        z = torch.from_numpy(uniform((n, H * D), seed=3)).to(dev)
        al = torch.from_numpy(uniform(H * D, seed=6)).to(dev)
        ar = torch.from_numpy(uniform(H * D, seed=7)).to(dev)
        for groups in (1, chunks):
            gt = RowPartitionedGAT(g, rank, world, H, D, head_groups=groups, device=dev,
                                   all_gather=None if backend == "nccl" else _staged_gather)
            gt.load_shard(z[gt.r0:gt.r1])
            yg = gt(al, ar)
            yr = torch.empty((n, H * D), device=dev)
            for h0, h1 in zip(gt.hg[:-1], gt.hg[1:]):
                zc = z[:, h0 * D:h1 * D].contiguous()
                el, er = G.gsp_attn_project(zc, al[h0 * D:h1 * D].contiguous(), ar[h0 * D:h1 * D].contiguous(),
                                            h1 - h0, D)
                yr[:, h0 * D:h1 * D] = G.gsp_gat_aggregate(g, el, er, zc, h1 - h0, D, 0.2)
            torch.cuda.synchronize()
            ok = ok and torch.equal(yg, yr[gt.r0:gt.r1])
        q.put((rank, ok, op.r0, op.r1))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), -1, -1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,backend,chunks", [(1, "nccl", 4), (2, "gloo", 1), (2, "gloo", 4), (3, "gloo", 2)])
def test_row_partitioned_spmm_on_one_gpu(world, backend, chunks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, backend, chunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    assert all(ok is True for _, ok, *_ in res), res
    assert res[0][2] == 0 and res[-1][3] == 20000
