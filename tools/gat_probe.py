"""Where does the fused GAT aggregate's time go?  C3 (Flickr-shaped, 8 x 64):
fused gsp_gat_aggregate vs gsp_multihead_spmm with a stored alpha (pure
aggregate) vs standalone gsp_edge_softmax (statistics + alpha), plus a
plain gsp_spmm of the same width.  L2 flushed before every timed call."""
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
z = torch.from_numpy(uniform((cfg.n, H * D), seed=3)).to(dev)
el = torch.from_numpy(uniform((cfg.n, H), seed=4, low=-3, high=3)).to(dev)
er = torch.from_numpy(uniform((cfg.n, H), seed=5, low=-3, high=3)).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
y = torch.empty((cfg.n, H * D), device=dev)
ws = torch.empty(max(G.gsp_gat_workspace(g, H), 16), dtype=torch.uint8, device=dev)
logits = torch.empty((g.nnz, H), device=dev)
_, alpha = G.gsp_gat_aggregate(g, el, er, z, H, D, 0.2, y=y, alpha_out=True, ws=ws)
logits.copy_(alpha)


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


res = {"workload": cfg.name, "nnz": g.nnz, "H": H, "D": D}
res["gat_aggregate_ms"] = t(lambda: G.gsp_gat_aggregate(g, el, er, z, H, D, 0.2, y=y, ws=ws))
res["gat_aggregate_single_launch_ms"] = t(lambda: G.gsp_gat_aggregate(g, el, er, z, H, D, 0.2, y=y,
                                                                      single_launch=True))
st = torch.empty((g.nnz, H), device=dev)
res["gat_row_stats_ms"] = t(lambda: G.gsp_edge_softmax(g, logits, H, alpha=st))
res["multihead_spmm_stored_alpha_ms"] = t(lambda: G.gsp_multihead_spmm(g, alpha, z, H, D, y=y))
res["edge_softmax_ms"] = t(lambda: G.gsp_edge_softmax(g, logits, H, alpha=logits))
res["spmm_512_ms"] = t(lambda: G.gsp_spmm(gn, z, f=H * D, y=y))
res["spmm_64_ms"] = t(lambda: G.gsp_spmm(gn, z[:, :64], f=64, y=y[:, :64]))
print(json.dumps(res))
