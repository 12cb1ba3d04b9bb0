"""C4 / C5: gsp_spmm (fp32 X) vs gsp_spmm_f16 (fp16 X, fp32 arithmetic), median ms, L2 flushed."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_00959_b200 as G  # noqa: E402
from synth import CONFIGS, features, graph_for  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


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


for key in sys.argv[1:] or ["C4", "C5"]:
    cfg = CONFIGS[key]
    s, d = graph_for(cfg, seed=1)
    g = G.gsp_sym_normalize(G.gsp_coo_to_csr(cfg.n, torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev),
                                             None, True, 1.0))
    f = cfg.f
    x = torch.from_numpy(features(cfg.n, f, cfg.ld, seed=2)).to(dev)
    ld16 = (f + 7) // 8 * 8
    xh = torch.zeros((cfg.n, ld16), dtype=torch.float16, device=dev)
    xh[:, :f] = x[:, :f].half()
    y = torch.empty((cfg.n, f), device=dev)
    r = {"config": key, "fp32_ms": t(lambda: G.gsp_spmm(g, x, f=f, y=y)),
         "f16_ms": t(lambda: G.gsp_spmm_f16(g, xh, f=f, y=y))}
    r["speedup"] = r["fp32_ms"] / r["f16_ms"]
    print(json.dumps(r), flush=True)
