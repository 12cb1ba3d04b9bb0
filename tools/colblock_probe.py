"""Does cutting A into column blocks (X row ranges) that fit L2 pay on C4?
Times the existing gsp_spmm on A restricted to each column block (same X,
same slab plan) against the full A.  Diagnostic only (no Y accumulation)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_00959_b200 as G  # noqa: E402
from synth import CONFIGS, features, graph_for  # noqa: E402

dev = torch.device("cuda", 0)
cfg = CONFIGS["C4"]
s, d = graph_for(cfg, seed=1)
s_t, d_t = torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev)
g = G.gsp_coo_to_csr(cfg.n, s_t, d_t, None, True, 1.0)
x = torch.from_numpy(features(cfg.n, cfg.f, cfg.ld, seed=2)).to(dev)
y = torch.empty((cfg.n, cfg.f), device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
# COO of A~ (symmetrised, self-loops) from the CSR
rows = torch.repeat_interleave(torch.arange(cfg.n, device=dev), g.row_ptr[1:] - g.row_ptr[:-1])
cols = g.col.long()


def t(a, slab=0, reps=10):
    for _ in range(3):
        G.gsp_spmm(a, x, f=cfg.f, y=y, slab_cols=slab)
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        G.gsp_spmm(a, x, f=cfg.f, y=y, slab_cols=slab)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


res = {"full_ms": t(g)}
for nb in (2, 4, 8):
    parts = []
    for b in range(nb):
        lo, hi = b * cfg.n // nb, (b + 1) * cfg.n // nb
        m = (cols >= lo) & (cols < hi)
        gb = G.gsp_coo_to_csr(cfg.n, rows[m].contiguous(), cols[m].contiguous(), None, False, 0.0)
        parts.append(t(gb))
        del gb
    res[f"blocks{nb}_ms_each"] = parts
    res[f"blocks{nb}_ms_sum"] = sum(parts)
for slab in (64, 128):
    res[f"full_slab{slab}_ms"] = t(g, slab)
print(json.dumps(res))
