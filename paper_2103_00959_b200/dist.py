"""Multi-GPU SpMM by row partition.

One process per GPU.  Every rank holds the full normalised CSR (built once,
replicated: normalisation needs remote degrees), owns the contiguous row block
[b_r, b_r+1) chosen by gsp_partition_rows (balanced by nnz), and keeps the
feature rows of exactly those nodes -- so Y's shard is the next layer's X
shard.  Per SpMM the only exchange is an equal-count all-gather of the padded
X shards (NCCL over NVLink/NVSwitch), after which the local slice (columns
remapped by gsp_csr_slice into the gathered layout) is multiplied by the
gathered X with the same kernel as on one GPU.  Because the kernel's
summation order depends only on the row, the P-GPU result is bitwise equal
to the 1-GPU result.

Overlap: the feature dimension is split into column chunks; the all-gather of
chunk c+1 (communication stream) runs while the SpMM of chunk c runs on the
compute stream.  Each chunk of the shard is stored contiguously
(chunk-packed) so every all-gather moves one contiguous buffer.

The collective is an abstract `all_gather(out, inp)` so the same driver runs
over NCCL (GPU) or gloo (CPU tests of the partition / layout logic).
"""
from __future__ import annotations

from typing import Callable, List, Optional

import torch

from . import (CSR, feature_ld, gsp_attn_project, gsp_csr_colblock, gsp_csr_slice, gsp_gat_aggregate,
               gsp_partition_rows, gsp_spmm, gsp_spmm_blocked)


class GpuOps:
    """The product's operators (libgsp kernels)."""

    @staticmethod
    def attn_project(z, a_l, a_r, heads, d, el, er):
        gsp_attn_project(z, a_l, a_r, heads, d, el=el, er=er)

    @staticmethod
    def gat_aggregate(local, el, er, z, heads, d, slope, y, ws):
        gsp_gat_aggregate(local, el, er, z, heads, d, slope, y=y, ws=ws)

    @staticmethod
    def partition(a, parts):
        return gsp_partition_rows(a, parts)[0]

    @staticmethod
    def slice(a, bounds, rank, npad):
        return gsp_csr_slice(a, bounds, rank, npad)

    @staticmethod
    def spmm(local, x, f, y):
        gsp_spmm(local, x, f=f, y=y)

    @staticmethod
    def colblock(local, bounds):
        return gsp_csr_colblock(local, bounds)

    @staticmethod
    def spmm_blocked(blocks, x, f, y):
        gsp_spmm_blocked(blocks, x, f=f, y=y)


def padded_rows(bounds: List[int]) -> int:
    return max(bounds[p + 1] - bounds[p] for p in range(len(bounds) - 1))


def remap_col_bounds(col_bounds: List[int], bounds: List[int], npad: int) -> List[int]:
    """Global column bounds -> the gathered layout's (gsp_csr_slice: column c
    of owner q -> q * npad + c - bounds[q]); the map is monotone, so a slice's
    block k holds exactly the global columns [col_bounds[k], col_bounds[k+1])."""
    world = len(bounds) - 1
    out = []
    for c in col_bounds:
        if c <= 0:
            out.append(0)
            continue
        if c >= bounds[world]:
            out.append(world * npad)
            continue
        q = max(p for p in range(world) if bounds[p] <= c < bounds[p + 1])  # the (non-empty) owner of c
        out.append(q * npad + (c - bounds[q]))
    return out


def chunk_bounds(f: int, chunks: int, align: int = 128) -> List[int]:
    """Column chunk edges, multiples of `align` (default: the 128-column slab
    width, so every chunk is whole slabs and needs no narrow tail launch)."""
    chunks = max(1, min(chunks, (f + align - 1) // align))
    step = ((f + chunks - 1) // chunks + align - 1) // align * align
    edges = list(range(0, f, step)) + [f]
    return edges


class RowPartitionedSpMM:
    """Y_shard = (A X)[rows of this rank] with X exchanged by all-gather."""

    def __init__(self, a: CSR, rank: int, world: int, f: int, chunks: int = 1,
                 all_gather: Optional[Callable] = None, device=None, ops=GpuOps, col_blocks=None):
        self.rank, self.world, self.f, self.ops = rank, world, f, ops
        self.bounds = [int(b) for b in ops.partition(a, world)]
        self.npad = padded_rows(self.bounds)
        self.r0, self.r1 = self.bounds[rank], self.bounds[rank + 1]
        self.rows = self.r1 - self.r0
        self.local = ops.slice(a, self.bounds, rank, self.npad)
        # column blocks (gsp_spmm_blocked): the GLOBAL bounds mapped into the
        # gathered layout, so each row's block partials and their sum are the
        # single-GPU gsp_spmm_blocked's (bitwise)
        self.col_blocks = None
        if col_blocks is not None and len(col_blocks) > 2 and self.rows:
            self.col_blocks = ops.colblock(self.local, remap_col_bounds(list(col_blocks), self.bounds, self.npad))
        self.cols = chunk_bounds(f, chunks)
        self.device = torch.device(device) if device is not None else a.row_ptr.device
        self.all_gather = all_gather or (lambda out, inp: torch.distributed.all_gather_into_tensor(out, inp))
        # chunk-packed shard and gathered buffers (each chunk contiguous; rows
        # padded to whole 128-byte lines, the library's feature layout)
        self.shard = [torch.zeros((self.npad, feature_ld(c1 - c0)), dtype=torch.float32, device=self.device)
                      for c0, c1 in zip(self.cols[:-1], self.cols[1:])]
        self.gathered = [torch.empty((world * self.npad, feature_ld(c1 - c0)), dtype=torch.float32,
                                     device=self.device) for c0, c1 in zip(self.cols[:-1], self.cols[1:])]
        self.comm = torch.cuda.Stream(device=self.device) if self.device.type == "cuda" else None

    def load_shard(self, x_rows: torch.Tensor):
        """x_rows: [rows, f] features of this rank's nodes."""
        for k, (c0, c1) in enumerate(zip(self.cols[:-1], self.cols[1:])):
            self.shard[k][:self.rows, :c1 - c0].copy_(x_rows[:, c0:c1])

    def exchange(self, k: int):
        self.all_gather(self.gathered[k], self.shard[k])

    def __call__(self, y: Optional[torch.Tensor] = None) -> torch.Tensor:
        if y is None:
            y = torch.empty((self.rows, self.f), dtype=torch.float32, device=self.device)
        nch = len(self.cols) - 1
        if self.comm is None:  # CPU / synchronous collectives
            for k in range(nch):
                self.exchange(k)
                self._local(k, y)
            return y
        main = torch.cuda.current_stream(self.device)
        self.comm.wait_stream(main)  # shard writes visible to the all-gather
        events = []
        with torch.cuda.stream(self.comm):
            for k in range(nch):
                self.exchange(k)
                ev = torch.cuda.Event()
                ev.record(self.comm)
                events.append(ev)
        for k in range(nch):
            main.wait_event(events[k])
            self._local(k, y)
        return y

    def _local(self, k: int, y: torch.Tensor):
        c0, c1 = self.cols[k], self.cols[k + 1]
        if self.rows and self.col_blocks is not None:
            self.ops.spmm_blocked(self.col_blocks, self.gathered[k][:, :c1 - c0], c1 - c0, y[:, c0:c1])
        elif self.rows:
            self.ops.spmm(self.local, self.gathered[k][:, :c1 - c0], c1 - c0, y[:, c0:c1])


class RowPartitionedPropagate(RowPartitionedSpMM):
    """y_shard = (sum_k theta_k A^k x)[rows of this rank] (K-step propagation,
    NEXT-4).  Step k all-gathers t_{k-1} (chunked, on the communication
    stream) and runs gsp_spmm_accumulate on the local slice, which writes t_k
    straight into this rank's shard buffers (the next step's all-gather
    source) and folds theta_k t_k into the local accumulator.  Bitwise equal
    to the single-GPU gsp_propagate (same per-element operations)."""

    def __call__(self, theta, y: Optional[torch.Tensor] = None) -> torch.Tensor:
        from . import gsp_spmm_accumulate
        K = len(theta) - 1
        if K < 1:
            raise ValueError("theta needs K >= 1 (len >= 2)")
        if y is None:
            y = torch.empty((self.rows, self.f), dtype=torch.float32, device=self.device)
        x0 = [s[:self.rows, :c1 - c0].clone() for s, c0, c1 in zip(self.shard, self.cols[:-1], self.cols[1:])]
        nch = len(self.cols) - 1
        for k in range(1, K + 1):
            def local(c):
                c0, c1 = self.cols[c], self.cols[c + 1]
                if self.rows:
                    gsp_spmm_accumulate(self.local, self.gathered[c][:, :c1 - c0], y[:, c0:c1], float(theta[k]),
                                        f=c1 - c0, t=self.shard[c][:self.rows, :c1 - c0] if k < K else None,
                                        src=x0[c] if k == 1 else None, src_coef=float(theta[0]))
            if self.comm is None:
                for c in range(nch):
                    self.exchange(c)
                    local(c)
                continue
            main = torch.cuda.current_stream(self.device)
            self.comm.wait_stream(main)  # previous step's t shard is complete
            events = []
            with torch.cuda.stream(self.comm):
                for c in range(nch):
                    self.exchange(c)
                    ev = torch.cuda.Event()
                    ev.record(self.comm)
                    events.append(ev)
            for c in range(nch):
                main.wait_event(events[c])
                local(c)
        return y


def head_chunks(heads: int, d: int, chunks: int, align: int = 128) -> List[int]:
    """Head-group edges for a chunked GAT exchange: every group is whole heads
    and, when possible, a multiple of `align` columns (whole 128-column slabs)."""
    chunks = max(1, min(chunks, heads))
    per = -(-heads // chunks)
    for p in range(per, heads + 1):
        if (p * d) % align == 0:
            per = p
            break
    return list(range(0, heads, per)) + [heads]


class RowPartitionedGAT:
    """Row-partitioned GAT aggregation ("GAT all-gathers Z
    (n x H.D) and er (n x H); el stays local").

    Each rank owns the row block [b_r, b_r+1) of the nnz-balanced partition and
    the Z rows of those nodes.  Per call it projects its own rows
    (gsp_attn_project -> el, er of its nodes), all-gathers er and Z over the
    padded equal-count layout (communication stream), keeps el local, and runs
    gsp_gat_aggregate on its CSR slice (columns remapped into the gathered
    layout by gsp_csr_slice).  Scores, softmax statistics and alpha of a row
    depend only on that row's el and its neighbours' er / Z, so with
    head_groups = 1 the result is bitwise equal to the single-GPU
    attn_project + gat_aggregate.  head_groups > 1 splits the heads into
    groups of whole heads so the all-gather of group g+1 overlaps the
    aggregate of group g (the statistics are then reduced per group: equal to
    the single-GPU call within the fp32 bound, not bitwise)."""

    def __init__(self, a: CSR, rank: int, world: int, heads: int, d: int, head_groups: int = 1,
                 negative_slope: float = 0.2, all_gather: Optional[Callable] = None, device=None, ops=GpuOps):
        self.rank, self.world, self.heads, self.d, self.ops = rank, world, heads, d, ops
        self.slope = negative_slope
        self.bounds = [int(b) for b in ops.partition(a, world)]
        self.npad = padded_rows(self.bounds)
        self.r0, self.r1 = self.bounds[rank], self.bounds[rank + 1]
        self.rows = self.r1 - self.r0
        self.local = ops.slice(a, self.bounds, rank, self.npad)
        self.hg = head_chunks(heads, d, head_groups)
        self.device = torch.device(device) if device is not None else a.row_ptr.device
        self.all_gather = all_gather or (lambda out, inp: torch.distributed.all_gather_into_tensor(out, inp))
        dv = self.device
        groups = list(zip(self.hg[:-1], self.hg[1:]))
        self.z_shard = [torch.zeros((self.npad, (h1 - h0) * d), dtype=torch.float32, device=dv) for h0, h1 in groups]
        self.er_shard = [torch.zeros((self.npad, h1 - h0), dtype=torch.float32, device=dv) for h0, h1 in groups]
        self.el = [torch.zeros((max(self.rows, 1), h1 - h0), dtype=torch.float32, device=dv) for h0, h1 in groups]
        self.z_all = [torch.empty((world * self.npad, (h1 - h0) * d), dtype=torch.float32, device=dv)
                      for h0, h1 in groups]
        self.er_all = [torch.empty((world * self.npad, h1 - h0), dtype=torch.float32, device=dv) for h0, h1 in groups]
        self.ws = None
        self.comm = torch.cuda.Stream(device=dv) if dv.type == "cuda" else None

    def load_shard(self, z_rows: torch.Tensor):
        """z_rows: [rows, H*D] features (after the layer's linear step) of this rank's nodes."""
        for k, (h0, h1) in enumerate(zip(self.hg[:-1], self.hg[1:])):
            self.z_shard[k][:self.rows].copy_(z_rows[:, h0 * self.d:h1 * self.d])

    def _project(self, k, a_l, a_r):
        h0, h1 = self.hg[k], self.hg[k + 1]
        if self.rows:
            self.ops.attn_project(self.z_shard[k][:self.rows], a_l[h0 * self.d:h1 * self.d].contiguous(),
                                  a_r[h0 * self.d:h1 * self.d].contiguous(), h1 - h0, self.d, self.el[k][:self.rows],
                                  self.er_shard[k][:self.rows])

    def _exchange(self, k):
        self.all_gather(self.er_all[k], self.er_shard[k])
        self.all_gather(self.z_all[k], self.z_shard[k])

    def _local(self, k, y):
        h0, h1 = self.hg[k], self.hg[k + 1]
        if self.rows:
            self.ops.gat_aggregate(self.local, self.el[k][:self.rows], self.er_all[k], self.z_all[k], h1 - h0, self.d,
                                   self.slope, y[:, h0 * self.d:h1 * self.d], self.ws)

    def __call__(self, a_l: torch.Tensor, a_r: torch.Tensor, y: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Y rows of this rank: [rows, H*D]; a_l, a_r: [H*D] attention vectors."""
        if y is None:
            y = torch.empty((self.rows, self.heads * self.d), dtype=torch.float32, device=self.device)
        ng = len(self.hg) - 1
        if self.comm is None:
            for k in range(ng):
                self._project(k, a_l, a_r)
                self._exchange(k)
                self._local(k, y)
            return y
        main = torch.cuda.current_stream(self.device)
        for k in range(ng):
            self._project(k, a_l, a_r)
        self.comm.wait_stream(main)  # er / Z shards complete before they are sent
        events = []
        with torch.cuda.stream(self.comm):
            for k in range(ng):
                self._exchange(k)
                ev = torch.cuda.Event()
                ev.record(self.comm)
                events.append(ev)
        for k in range(ng):
            main.wait_event(events[k])
            self._local(k, y)
        return y
