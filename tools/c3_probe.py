"""Why is the C3 (Flickr-shaped, 8 x 64) aggregate slower per gathered byte
than C4's SpMM?  Times, with L2 flushed before every call:
  * the fused GAT, the multi-head SpMM with stored alpha, plain gsp_spmm at
    F = 512 on the same graph (weight policy cost);
  * gsp_spmm at F = 512 with row-block sizes 1024 .. 16384 (tail / CTA
    prologue cost) and slab widths 64 / 128;
  * the same graph with every row's degree histogram printed (short rows)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_00959_b200 as G  # noqa: E402
from synth import CONFIGS, graph_for, uniform  # noqa: E402

dev = torch.device("cuda", 0)
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
H, D = 8, 64
s, d = graph_for(cfg, seed=1)
g = G.gsp_coo_to_csr(cfg.n, torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev), None, True, 1.0)
gn = G.gsp_sym_normalize(g)
F = H * D
z = G.empty_features(cfg.n, F, dev)
z[:, :F] = torch.from_numpy(uniform((cfg.n, F), seed=3)).to(dev)
el = torch.from_numpy(uniform((cfg.n, H), seed=4, low=-3, high=3)).to(dev)
er = torch.from_numpy(uniform((cfg.n, H), seed=5, low=-3, high=3)).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
y = G.empty_features(cfg.n, F, dev)
ws = torch.empty(max(G.gsp_gat_workspace(g, H), 16), dtype=torch.uint8, device=dev)
_, alpha = G.gsp_gat_aggregate(g, el, er, z, H, D, 0.2, y=y, alpha_out=True, ws=ws)


def t(fn, reps=20):
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
    return float(np.median(ts))


rp = g.row_ptr.cpu().numpy()
deg = np.diff(rp)
res = {"workload": cfg.name, "n": cfg.n, "nnz": g.nnz,
       "deg_pct_10_25_50_75_90_99": np.percentile(deg, [10, 25, 50, 75, 90, 99]).tolist(),
       "rows_le4": int((deg <= 4).sum()), "rows_le8": int((deg <= 8).sum()),
       "nnz_frac_rows_le8": float(deg[deg <= 8].sum() / deg.sum()),
       "nnz_frac_rows_gt512": float(deg[deg > 512].sum() / deg.sum())}
res["gat_fused_ms"] = t(lambda: G.gsp_gat_aggregate(g, el, er, z, H, D, 0.2, y=y, ws=ws))
res["multihead_stored_alpha_ms"] = t(lambda: G.gsp_multihead_spmm(g, alpha, z, H, D, y=y))
res["spmm_512_ms"] = t(lambda: G.gsp_spmm(gn, z, f=F, y=y))
for b in (1024, 2048, 4096, 8192, 16384):
    res[f"spmm_512_block{b}_ms"] = t(lambda: G.gsp_spmm(gn, z, f=F, y=y, block_nnz=b))
res["spmm_512_slab64_ms"] = t(lambda: G.gsp_spmm(gn, z, f=F, y=y, slab_cols=64))
res["spmm_128_ms"] = t(lambda: G.gsp_spmm(gn, z, f=128, y=y))
ge = g.nnz * F
for k in list(res):
    if k.endswith("_ms") and "spmm" in k:
        res[k.replace("_ms", "_TBs_gather")] = ge * 4 / (res[k] * 1e-3) / 1e12 if "128" not in k else None
print(json.dumps(res))
