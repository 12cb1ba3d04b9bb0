"""Row alignment of X vs L2 capacity: gsp_spmm on C4 / C5 with X row strides
ld = round_up(F, 4) (16-byte rows) and ld = round_up(F, 32) (128-byte rows,
every row-slab whole L2 lines), for the default and narrower slabs.  L2
flushed before every timed call; results bitwise equal across ld / slabs."""
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
    return float(np.median(ts))


res = {}
for key in (sys.argv[1:] or ["C4", "C5"]):
    cfg = CONFIGS[key]
    s, d = graph_for(cfg, seed=1)
    gn = G.gsp_sym_normalize(G.gsp_coo_to_csr(cfg.n, torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev)))
    f = cfg.f
    x0 = torch.from_numpy(features(cfg.n, f, f, seed=2)).to(dev)
    yref = None
    lds = [int(v) for v in os.environ.get("LDS", "").split(",") if v] or \
        sorted({(f + 3) // 4 * 4, (f + 31) // 32 * 32, (f + 63) // 64 * 64})
    slabs = [int(v) for v in os.environ.get("SLABS", "0,64,32").split(",")]
    for ld in lds:
        buf = torch.zeros((cfg.n, ld), device=dev)
        buf[:, :f] = x0
        x = buf[:, :f]
        for slab in slabs:
            y = torch.empty((cfg.n, f), device=dev)
            ms = t(lambda: G.gsp_spmm(gn, x, f=f, y=y, slab_cols=slab))
            if yref is None:
                yref = y.clone()
            res[f"{key} ld={ld} slab={slab or 'auto'}"] = {"ms": ms, "GE/s": gn.nnz * f / (ms * 1e-3),
                                                          "bitwise_equal": bool(torch.equal(y, yref))}
            print(key, ld, slab, ms, flush=True)
        x16 = torch.zeros((cfg.n, ld), dtype=torch.float16, device=dev)
        x16[:, :f] = x0.half()
        y = torch.empty((cfg.n, f), device=dev)
        res[f"{key} f16 ld={ld}"] = {"ms": t(lambda: G.gsp_spmm_f16(gn, x16[:, :f], f=f, y=y))}
        del buf, x16
print(json.dumps(res, indent=1))
