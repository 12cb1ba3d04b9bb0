"""racecheck probe: single-launch GAT aggregate with / without hub rows (argv[1] = hubs|nohubs)."""
import sys
import numpy as np
import torch
import paper_2103_00959_b200 as G
from synth import chung_lu, uniform

dev = torch.device("cuda", 0)
n, m = 3000, 25000
s, d = chung_lu(n, m, seed=3)
if sys.argv[1] == "hubs":
    s = np.concatenate([s, np.zeros(1500, np.int64)])
    d = np.concatenate([d, np.arange(1, 1501, dtype=np.int64)])
g = G.gsp_coo_to_csr(n, torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev))
H, D = 8, 16
z = torch.from_numpy(uniform((n, H * D), seed=1)).to(dev)
el = torch.from_numpy(uniform((n, H), seed=2)).to(dev)
er = torch.from_numpy(uniform((n, H), seed=3)).to(dev)
G.gsp_gat_aggregate(g, el, er, z, H, D, single_launch=True)
torch.cuda.synchronize()
print("ok", int((g.row_ptr[1:] - g.row_ptr[:-1]).max()))
