"""a2 (gsp_sym_normalize) on C4 / C5: median ms with L2 flushed, and a checksum
of the normalised values (variants must agree bit for bit)."""
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
    g = G.gsp_coo_to_csr(cfg.n, torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev))
    gn = G.gsp_sym_normalize(g)
    ts = []
    for i in range(13):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); gn = G.gsp_sym_normalize(g); b.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(a.elapsed_time(b))
    res[key + "_ms"] = round(float(np.median(ts)), 4)
    res[key + "_sha"] = hashlib.sha1(gn.val.cpu().numpy().tobytes() + gn.deg.cpu().numpy().tobytes()).hexdigest()[:12]
print(json.dumps(res))
