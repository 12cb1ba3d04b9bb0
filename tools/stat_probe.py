"""Row statistics variants on C3 (8 x 64): fused GAT and standalone edge
softmax, median ms with L2 flushed, and checksums of the outputs (variants
must agree bit for bit)."""
import hashlib, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_00959_b200 as G  # noqa: E402
from synth import CONFIGS, graph_for, uniform  # noqa: E402
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res = {"lib": os.path.basename(G.LIB_PATH)}
for key in sys.argv[1:] or ["C3", "C2g"]:
    cfg = CONFIGS[key]
    H, D = 8, 64
    s, d = graph_for(cfg, seed=1)
    g = G.gsp_coo_to_csr(cfg.n, torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev))
    z = G.empty_features(cfg.n, H * D, dev)
    z[:, :H * D] = torch.from_numpy(uniform((cfg.n, H * D), seed=3)).to(dev)
    el = torch.from_numpy(uniform((cfg.n, H), seed=4, low=-3, high=3)).to(dev)
    er = torch.from_numpy(uniform((cfg.n, H), seed=5, low=-3, high=3)).to(dev)
    y = G.empty_features(cfg.n, H * D, dev)
    ws = torch.empty(G.gsp_gat_workspace(g, H), dtype=torch.uint8, device=dev)
    lg = torch.from_numpy(uniform((g.nnz, H), seed=6, low=-4, high=4)).to(dev)
    al = torch.empty_like(lg)

    def t(fn):
        ts = []
        for i in range(23):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); torch.cuda.synchronize()
            if i >= 3: ts.append(a.elapsed_time(b))
        return round(float(np.median(ts)), 4)
    res[key + "_gat_ms"] = t(lambda: G.gsp_gat_aggregate(g, el, er, z, H, D, 0.2, y=y, ws=ws))
    res[key + "_gat_sha"] = hashlib.sha1(y.cpu().numpy().tobytes()).hexdigest()[:12]
    res[key + "_softmax_ms"] = t(lambda: G.gsp_edge_softmax(g, lg, H, alpha=al))
    res[key + "_softmax_sha"] = hashlib.sha1(al.cpu().numpy().tobytes()).hexdigest()[:12]
print(json.dumps(res))
