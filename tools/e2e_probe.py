"""HostSpMM (pinned host X -> device -> gsp_spmm -> host Y) on C4 for several copy-slab widths (median ms)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_00959_b200 as G  # noqa: E402
from paper_2103_00959_b200.host import HostSpMM  # noqa: E402
from synth import CONFIGS, features, graph_for  # noqa: E402

dev = torch.device("cuda", 0)
cfg = CONFIGS["C4"]
s, d = graph_for(cfg, seed=1)
g = G.gsp_sym_normalize(G.gsp_coo_to_csr(cfg.n, torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev), None,
                                         True, 1.0))
xh = torch.from_numpy(features(cfg.n, cfg.f, cfg.ld, seed=2)).pin_memory()
yh = torch.empty((cfg.n, cfg.ld), dtype=torch.float32).pin_memory()
res = {}
for slab in [int(v) for v in (sys.argv[1:] or ["128", "256", "192", "384", "64"])]:
    hs = HostSpMM(g, cfg.f, cfg.ld, slab=slab, device=dev)
    ts = []
    for i in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        hs(xh, yh)
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    res[slab] = float(np.median(ts))
    del hs
print(json.dumps(res))
