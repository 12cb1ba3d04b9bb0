"""Time one libgsp build (GSP_LIB=path, else the in-tree one) on the headline
kernels: C4 / C5 SpMM in the library's feature layout, the C3 fused GAT
aggregate and its statistics launch (edge softmax), L2 flushed before every
call.  Prints one JSON line.  Usage: GSP_LIB=variants/libgsp_x.so python tools/variant_probe.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_00959_b200 as G  # noqa: E402
from synth import CONFIGS, features, graph_for, uniform  # noqa: E402

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


res = {"lib": os.path.basename(G.LIB_PATH)}
which = sys.argv[1:] or ["C4", "C5", "C3"]
for key in which:
    cfg = CONFIGS[key]
    s, d = graph_for(cfg, seed=1)
    g = G.gsp_coo_to_csr(cfg.n, torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev))
    if cfg.heads == 1:
        gn = G.gsp_sym_normalize(g)
        x = G.empty_features(cfg.n, cfg.f, dev)
        x.copy_(torch.from_numpy(features(cfg.n, cfg.f, cfg.f, seed=2)))
        y = G.empty_features(cfg.n, cfg.f, dev)
        res[f"{key}_spmm_ms"] = t(lambda: G.gsp_spmm(gn, x, f=cfg.f, y=y))
    else:
        H, D = cfg.heads, cfg.d
        z = torch.from_numpy(uniform((cfg.n, H * D), seed=3)).to(dev)
        el = torch.from_numpy(uniform((cfg.n, H), seed=4, low=-3, high=3)).to(dev)
        er = torch.from_numpy(uniform((cfg.n, H), seed=5, low=-3, high=3)).to(dev)
        y = G.empty_features(cfg.n, H * D, dev)
        ws = torch.empty(G.gsp_gat_workspace(g, H), dtype=torch.uint8, device=dev)
        _, alpha = G.gsp_gat_aggregate(g, el, er, z, H, D, 0.2, y=y, alpha_out=True, ws=ws)
        lg = alpha.clone()
        res[f"{key}_gat_ms"] = t(lambda: G.gsp_gat_aggregate(g, el, er, z, H, D, 0.2, y=y, ws=ws))
        res[f"{key}_softmax_ms"] = t(lambda: G.gsp_edge_softmax(g, lg, H, alpha=alpha))
        res[f"{key}_multihead_ms"] = t(lambda: G.gsp_multihead_spmm(g, alpha, z, H, D, y=y))
    del g
    torch.cuda.empty_cache()
print(json.dumps(res), flush=True)
