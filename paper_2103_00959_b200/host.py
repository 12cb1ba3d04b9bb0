"""SpMM from/to HOST buffers with the copies pipelined against the kernel.

gsp_spmm gathers X rows at random, so no output row is final before all of X
has arrived -- but a column slab of Y depends only on the same column slab of
X.  The call is therefore cut into column slabs (multiples of the 128-column
engine slab): the H2D copy of slab s+1 (copy stream), the SpMM of slab s
(compute stream) and the D2H copy of slab s-1 (second copy stream) run
concurrently; PCIe is full duplex, so the step costs about
max(H2D bytes, D2H bytes) / link bandwidth plus one slab of compute.

Orchestration only (streams, events, strided cudaMemcpy2DAsync DMA through
cuda-python); every arithmetic step is gsp_spmm in libgsp.
"""
from __future__ import annotations

from typing import List

import torch
from cuda.bindings import runtime as _rt

from . import CSR, gsp_spmm, gsp_spmm_blocked


def _copy2d(dst: torch.Tensor, src: torch.Tensor, kind, stream: torch.cuda.Stream):
    """Strided 2-D copy of a [rows, cols] fp32 view (unit column stride) by DMA."""
    rows, cols = src.shape
    err, = _rt.cudaMemcpy2DAsync(dst.data_ptr(), dst.stride(0) * 4, src.data_ptr(), src.stride(0) * 4, cols * 4,
                                 rows, kind, stream.cuda_stream)
    if err != _rt.cudaError_t.cudaSuccess:
        raise RuntimeError(f"cudaMemcpy2DAsync failed: {err}")


class HostSpMM:
    """y_host[:, :f] = A @ x_host[:, :f] with pinned host x_host, y_host."""

    def __init__(self, a: CSR, f: int, ld: int, slab: int = 128, device=None, blocks=None):
        self.a, self.f, self.ld, self.blocks = a, f, ld, blocks
        self.device = torch.device(device) if device is not None else a.row_ptr.device
        self.cols: List[int] = list(range(0, f, slab)) + [f]
        self.x = torch.empty((a.n_cols, ld), dtype=torch.float32, device=self.device)
        self.y = torch.empty((a.n_rows, ld), dtype=torch.float32, device=self.device)
        self.h2d = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)

    def __call__(self, x_host: torch.Tensor, y_host: torch.Tensor):
        main = torch.cuda.current_stream(self.device)
        ns = len(self.cols) - 1
        loaded = [torch.cuda.Event() for _ in range(ns)]
        done = [torch.cuda.Event() for _ in range(ns)]
        self.h2d.wait_stream(main)
        with torch.cuda.stream(self.h2d):
            for s in range(ns):
                c0, c1 = self.cols[s], self.cols[s + 1]
                _copy2d(self.x[:, c0:c1], x_host[:, c0:c1], _rt.cudaMemcpyKind.cudaMemcpyHostToDevice, self.h2d)
                loaded[s].record(self.h2d)
        for s in range(ns):
            c0, c1 = self.cols[s], self.cols[s + 1]
            main.wait_event(loaded[s])
            if self.blocks is not None:  # column blocks of A (gsp_csr_colblock)
                gsp_spmm_blocked(self.blocks, self.x[:, c0:c1], f=c1 - c0, y=self.y[:, c0:c1])
            else:
                gsp_spmm(self.a, self.x[:, c0:c1], f=c1 - c0, y=self.y[:, c0:c1])
            done[s].record(main)
        with torch.cuda.stream(self.d2h):
            for s in range(ns):
                c0, c1 = self.cols[s], self.cols[s + 1]
                self.d2h.wait_event(done[s])
                _copy2d(y_host[:, c0:c1], self.y[:, c0:c1], _rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, self.d2h)
        main.wait_stream(self.d2h)
        return y_host

    def launches(self) -> int:
        from . import gsp_spmm_plan_info
        mats = [self.blocks.block(k) for k in range(len(self.blocks))] if self.blocks is not None else [self.a]
        return sum(gsp_spmm_plan_info(m, self.x[:, c0:c1], c1 - c0)[0]
                   for m in mats for c0, c1 in zip(self.cols[:-1], self.cols[1:]))
