#!/usr/bin/env python
"""Driver for the per-(config, op) ncu pass behind bench.py's report rows.

Builds the bench's inputs (same generators, seeds and shapes) and calls every
(config, op) of the report ONCE inside an NVTX push/pop range named
"ncu|<workload>|<op>".  Run it under

  ncu --nvtx --print-nvtx-rename kernel --clock-control none --cache-control all \
      --metrics <list> --csv --log-file gpurun_out/ncu_ops.csv python tools/ncu_ops.py

so every profiled launch of an op carries the op's name; tools/ncu_rows.py
then sums the launches of each op into profiles/<tag>_ncu_rows.json, which
bench.py joins into its rows (ncu DRAM bytes, L2 hit rate).  ncu's
--cache-control all flushes the caches before each launch, matching the
bench's cold (L2-flushed) timing.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_00959_b200 as G  # noqa: E402
from synth import CONFIGS, features, graph_for, uniform  # noqa: E402

dev = torch.device("cuda", 0)


def rng(name):
    class R:
        def __enter__(self):
            torch.cuda.synchronize()
            torch.cuda.nvtx.range_push(name)

        def __exit__(self, *a):
            torch.cuda.synchronize()
            torch.cuda.nvtx.range_pop()
    return R()


def build(key):
    cfg = CONFIGS[key]
    s, d = graph_for(cfg, seed=1)
    st, dt = torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev)
    return cfg, st, dt


def gcn(key, with_build=False):
    cfg, st, dt = build(key)
    if with_build:
        G.gsp_coo_to_csr(cfg.n, st, dt, None, True, 1.0)  # first call (allocator / attributes)
        with rng(f"ncu|{cfg.name}|a1_build"):
            g = G.gsp_coo_to_csr(cfg.n, st, dt, None, True, 1.0)
        G.gsp_sym_normalize(g)
        with rng(f"ncu|{cfg.name}|a2_normalize"):
            gn = G.gsp_sym_normalize(g)
    else:
        g = G.gsp_coo_to_csr(cfg.n, st, dt, None, True, 1.0)
        gn = G.gsp_sym_normalize(g)
    del st, dt
    x = G.empty_features(cfg.n, cfg.f, dev)
    x.copy_(torch.from_numpy(features(cfg.n, cfg.f, cfg.f, seed=2)))
    y = G.empty_features(cfg.n, cfg.f, dev)
    G.gsp_spmm(gn, x, f=cfg.f, y=y)
    with rng(f"ncu|{cfg.name}|a3_spmm"):
        G.gsp_spmm(gn, x, f=cfg.f, y=y)
    bounds = G.colblock_bounds(gn, cfg.f)
    if len(bounds) > 2:  # bench.py's headline plan (column blocks)
        blocks = G.gsp_csr_colblock(gn, bounds)
        G.gsp_spmm_blocked(blocks, x, f=cfg.f, y=y)
        with rng(f"ncu|{cfg.name}|a3_spmm_colblocked"):
            G.gsp_spmm_blocked(blocks, x, f=cfg.f, y=y)


def gat(key, H, D):
    cfg, st, dt = build(key)
    name = f"{cfg.name.split('-gat')[0]}-gat{H}x{D}"
    g = G.gsp_coo_to_csr(cfg.n, st, dt, None, True, 1.0)
    z = torch.from_numpy(uniform((cfg.n, H * D), seed=3)).to(dev)
    al = torch.from_numpy(uniform((H, D), seed=6).reshape(-1)).to(dev)
    ar = torch.from_numpy(uniform((H, D), seed=7).reshape(-1)).to(dev)
    el, er = G.gsp_attn_project(z, al, ar, H, D)
    y = torch.empty((cfg.n, H * D), dtype=torch.float32, device=dev)
    ws = torch.empty(G.gsp_gat_workspace(g, H), dtype=torch.uint8, device=dev)
    with rng(f"ncu|{name}|a4_attn_project"):
        G.gsp_attn_project(z, al, ar, H, D, el=el, er=er)
    G.gsp_gat_aggregate(g, el, er, z, H, D, 0.2, y=y, ws=ws)
    with rng(f"ncu|{name}|a5-a7_gat_fused"):
        G.gsp_gat_aggregate(g, el, er, z, H, D, 0.2, y=y, ws=ws)
    _, alpha = G.gsp_gat_aggregate(g, el, er, z, H, D, 0.2, y=y, alpha_out=True, ws=ws)
    logits = alpha.clone()
    with rng(f"ncu|{name}|a6_edge_softmax"):
        G.gsp_edge_softmax(g, logits, H, alpha=alpha)
    with rng(f"ncu|{name}|a7_multihead_spmm"):
        G.gsp_multihead_spmm(g, alpha, z, H, D, y=y)


def main():
    which = sys.argv[1:] or ["C4", "C1", "C2", "C5", "C2g8", "C2g64", "C3"]
    for w in which:
        if w in ("C1", "C2", "C5", "C6"):
            gcn(w)
        elif w == "C4":
            gcn("C4", with_build=True)
        elif w == "C2g8":
            gat("C2g", 8, 8)
        elif w == "C2g64":
            gat("C2g", 8, 64)
        elif w == "C3":
            gat("C3", 8, 64)
        torch.cuda.empty_cache()
    print("ncu_ops done")


if __name__ == "__main__":
    main()
