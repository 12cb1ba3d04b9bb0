"""Probe: C4 / C5 SpMM as K column blocks of A (X row ranges of n/K rows):
Y = A_0 X_0, then Y += A_k X_k (gsp_spmm_accumulate, coef 1) -- each launch
gathers from a K-times smaller X footprint per slab.  The blocks are separate
CSR objects built here with torch (a probe, not the product path).  Median ms
with L2 flushed; the result is checked against the one-launch SpMM within the
fp32 bound (the summation order differs)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_00959_b200 as G  # noqa: E402
from synth import CONFIGS, features, graph_for  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def t(fn, reps=15):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return round(float(np.median(ts)), 4)


def col_blocks(g, k):
    n = g.n_cols
    rows = torch.repeat_interleave(torch.arange(g.n_rows, device=dev), torch.diff(g.row_ptr))
    out = []
    for b in range(k):
        lo, hi = b * n // k, (b + 1) * n // k
        m = (g.col >= lo) & (g.col < hi)
        rp = torch.zeros(g.n_rows + 1, dtype=torch.int64, device=dev)
        rp[1:] = torch.cumsum(torch.bincount(rows[m], minlength=g.n_rows), 0)
        out.append(G.CSR(rp, g.col[m].contiguous(), g.val[m].contiguous(), n))
    return out


res = {}
for key in (sys.argv[1:] or ["C4", "C5"]):
    cfg = CONFIGS[key]
    s, d = graph_for(cfg, seed=1)
    gn = G.gsp_sym_normalize(G.gsp_coo_to_csr(cfg.n, torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev)))
    f = cfg.f
    x = G.empty_features(cfg.n, f, dev)
    x.copy_(torch.from_numpy(features(cfg.n, f, f, seed=2)))
    y = G.empty_features(cfg.n, f, dev)
    res[f"{key} one launch"] = t(lambda: G.gsp_spmm(gn, x, f=f, y=y))
    yref = y.clone()
    absx = x.abs()
    cond = G.gsp_spmm(G.CSR(gn.row_ptr, gn.col, gn.val.abs(), gn.n_cols), absx, f=f)
    for k in (2, 3, 4):
        blocks = col_blocks(gn, k)

        def run():
            G.gsp_spmm(blocks[0], x, f=f, y=y)
            for bl in blocks[1:]:
                G.gsp_spmm_accumulate(bl, x, y, 1.0, f=f)
        ms = t(run)
        err = ((y[:, :f] - yref[:, :f]).abs() / (1e-5 * cond[:, :f] + 1e-6)).max().item()
        res[f"{key} {k} column blocks"] = {"ms": ms, "max_err_over_bound_vs_one_launch": round(err, 4)}
        print(key, k, ms, err, flush=True)
        del blocks
    del gn, x, y, yref, cond
    torch.cuda.empty_cache()
print(json.dumps(res, indent=1))
