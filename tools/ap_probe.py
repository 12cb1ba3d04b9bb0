"""gsp_attn_project on C3 (8 x 64): median ms, L2 flushed."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_00959_b200 as G  # noqa: E402
from synth import CONFIGS, uniform  # noqa: E402
dev = torch.device("cuda", 0)
cfg = CONFIGS["C3"]
H, D = 8, 64
z = torch.from_numpy(uniform((cfg.n, H * D), seed=3)).to(dev)
al = torch.from_numpy(uniform(H * D, seed=6)).to(dev)
ar = torch.from_numpy(uniform(H * D, seed=7)).to(dev)
el, er = G.gsp_attn_project(z, al, ar, H, D)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
mode = sys.argv[1] if len(sys.argv) > 1 else "write"
ts = []
for i in range(23):
    if mode == "write":
        flush.zero_()  # the bench's flush: leaves 256 MB of dirty lines in L2
    else:
        flush.max()  # read-only flush: evicts without dirty lines
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); G.gsp_attn_project(z, al, ar, H, D, el=el, er=er); b.record(); torch.cuda.synchronize()
    if i >= 3: ts.append(a.elapsed_time(b))
print(json.dumps({"flush": mode, "attn_project_ms": float(np.median(ts)), "GB/s": (z.numel() * 4 + 2 * el.numel() * 4) / (np.median(ts) * 1e-3) / 1e9}))
