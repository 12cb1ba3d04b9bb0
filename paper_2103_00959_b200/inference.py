"""2-layer GCN and GAT inference (NEXT-1) composed from the C-ABI calls.

The workload of the paper's Table spmm_time: "end-to-end inference
time ... of 2-layer GCN and GAT models with hidden size 128; the GAT model uses
4 attention heads" (reading A20: 4 heads x 32 = 128 hidden, ELU on the hidden
layer, one output head -- the standard GAT arrangement).

    GCN (Eq. gcn_layer):  H1 = ReLU(A^ (X W1) + b1);  Y = A^ (H1 W2) + b2
    GAT:      Z = X W1; el, er = Z a_l, Z a_r;
                                 H1 = ELU(GATAggregate(Z) + b1);  second layer likewise, 1 head

Every arithmetic step runs in libgsp (cuBLAS for the dense X W, the SpMM
engine for aggregation + bias + activation); this module only orders the
calls and holds the (random-init, seeded) parameters.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import (CSR, empty_features, gsp_attn_project, gsp_gat_aggregate_bias_act, gsp_gcn_layer, gsp_linear)


def _padded(n: int, cols: int, device) -> torch.Tensor:
    """[n, cols] view of a buffer in the library's feature layout (rows on
    whole 128-byte lines, padding columns zeroed: the next layer's gathers may
    read them and they stay defined) -- gsp.h, DESIGN.md §2."""
    return empty_features(n, cols, device)


def _glorot(shape, rng):
    lim = np.sqrt(6.0 / (shape[0] + shape[-1]))
    return (rng.uniform(-lim, lim, shape)).astype(np.float32)


@dataclass
class GCNParams:
    w1: torch.Tensor
    b1: torch.Tensor
    w2: torch.Tensor
    b2: torch.Tensor

    @staticmethod
    def init(f_in, hidden, classes, device, seed=0):
        rng = np.random.default_rng(seed)
        t = lambda a: torch.from_numpy(a).to(device)
        return GCNParams(t(_glorot((f_in, hidden), rng)), t(np.zeros(hidden, np.float32)),
                         t(_glorot((hidden, classes), rng)), t(np.zeros(classes, np.float32)))


def gcn_inference(a: CSR, x: torch.Tensor, p: GCNParams) -> torch.Tensor:
    """Two GCN layers on the normalised adjacency a (2 GEMM + 2 SpMM launches)."""
    h1 = gsp_gcn_layer(a, x, p.w1, p.b1, "relu", y=_padded(a.n_rows, p.w1.shape[1], x.device))
    return gsp_gcn_layer(a, h1, p.w2, p.b2, "none", y=_padded(a.n_rows, p.w2.shape[1], x.device))


@dataclass
class GATParams:
    w1: torch.Tensor
    al1: torch.Tensor
    ar1: torch.Tensor
    b1: torch.Tensor
    w2: torch.Tensor
    al2: torch.Tensor
    ar2: torch.Tensor
    b2: torch.Tensor
    heads1: int
    d1: int
    classes: int

    @staticmethod
    def init(f_in, hidden, heads, classes, device, seed=0):
        rng = np.random.default_rng(seed)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)
        d1 = hidden // heads
        return GATParams(t(_glorot((f_in, hidden), rng)), t(_glorot((heads, d1), rng).reshape(-1)),
                         t(_glorot((heads, d1), rng).reshape(-1)), t(np.zeros(hidden, np.float32)),
                         t(_glorot((hidden, classes), rng)), t(_glorot((1, classes), rng).reshape(-1)),
                         t(_glorot((1, classes), rng).reshape(-1)), t(np.zeros(classes, np.float32)),
                         heads, d1, classes)


def gat_inference(a: CSR, x: torch.Tensor, p: GATParams, negative_slope: float = 0.2) -> torch.Tensor:
    """Two GAT layers on the self-looped graph a (values unused)."""
    dev = x.device
    z1 = gsp_linear(x, p.w1, y=_padded(a.n_cols, p.w1.shape[1], dev))
    el1, er1 = gsp_attn_project(z1, p.al1, p.ar1, p.heads1, p.d1)
    h1 = gsp_gat_aggregate_bias_act(a, el1, er1, z1, p.heads1, p.d1, p.b1, "elu", negative_slope,
                                    y=_padded(a.n_rows, p.heads1 * p.d1, dev))
    z2 = gsp_linear(h1, p.w2, y=_padded(a.n_cols, p.classes, dev))
    el2, er2 = gsp_attn_project(z2, p.al2, p.ar2, 1, p.classes)
    return gsp_gat_aggregate_bias_act(a, el2, er2, z2, 1, p.classes, p.b2, "none", negative_slope,
                                      y=_padded(a.n_rows, p.classes, dev))
