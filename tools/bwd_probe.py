"""NEXT-3 kernels on C3 (8 x 64): SDDMM, edge-softmax backward, full GAT aggregate backward (median ms)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_00959_b200 as G  # noqa: E402
from synth import CONFIGS, graph_for, uniform  # noqa: E402

dev = torch.device("cuda", 0)
cfg = CONFIGS["C3"]
H, D = 8, 64
s, d = graph_for(cfg, seed=1)
g = G.gsp_coo_to_csr(cfg.n, torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev), None, True, 1.0)
z = torch.from_numpy(uniform((cfg.n, H * D), seed=3)).to(dev)
el = torch.from_numpy(uniform((cfg.n, H), seed=4, low=-3, high=3)).to(dev)
er = torch.from_numpy(uniform((cfg.n, H), seed=5, low=-3, high=3)).to(dev)
dy = torch.from_numpy(uniform((cfg.n, H * D), seed=6)).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
_, alpha = G.gsp_gat_aggregate(g, el, er, z, H, D, alpha_out=True)
at, perm = G.gsp_csr_transpose(g)
buf = torch.empty_like(alpha)


def t(fn, reps=10):
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


print(json.dumps({"sddmm_ms": t(lambda: G.gsp_sddmm(g, dy, z, heads=H, out=buf)),
                  "softmax_bwd_ms": t(lambda: G.gsp_edge_softmax_backward(g, alpha, buf, H, ds=buf)),
                  "gat_bwd_ms": t(lambda: G.gsp_gat_aggregate_backward(g, at, perm, el, er, z, dy, H, D), 5)}))
