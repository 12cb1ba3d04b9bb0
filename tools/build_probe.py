"""a1 (gsp_coo_to_csr) on C4 / C5: median ms with L2 flushed, and a checksum
of the CSR (variants must agree bit for bit)."""
import hashlib, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_00959_b200 as G  # noqa: E402
from synth import CONFIGS, graph_for  # noqa: E402
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res = {"lib": os.path.basename(G.LIB_PATH)}
for key in sys.argv[1:] or ["C4", "C5"]:
    cfg = CONFIGS[key]
    s, d = graph_for(cfg, seed=1)
    src, dst = torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev)
    g = G.gsp_coo_to_csr(cfg.n, src, dst, None, True, 1.0)
    ts = []
    for i in range(13):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g = G.gsp_coo_to_csr(cfg.n, src, dst, None, True, 1.0); b.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(a.elapsed_time(b))
    res[key + "_ms"] = round(float(np.median(ts)), 4)
    h = hashlib.sha1(g.row_ptr.cpu().numpy().tobytes() + g.col.cpu().numpy().tobytes() + g.val.cpu().numpy().tobytes())
    res[key + "_sha"] = h.hexdigest()[:12]
print(json.dumps(res))
