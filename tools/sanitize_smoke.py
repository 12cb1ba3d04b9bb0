"""Small calls of every libgsp operator, for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck).  Exits non-zero on a status error."""
import numpy as np
import torch

import paper_2103_00959_b200 as G
from paper_2103_00959_b200.inference import GATParams, GCNParams, gat_inference, gcn_inference
from synth import chung_lu, features, uniform

dev = torch.device("cuda", 0)
n, m = 3000, 25000
s, d = chung_lu(n, m, seed=3)
# hub rows so the CTA-cooperative path runs too
s = np.concatenate([s, np.zeros(1500, np.int64)])
d = np.concatenate([d, np.arange(1, 1501, dtype=np.int64)])
g = G.gsp_coo_to_csr(n, torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev))
gn = G.gsp_sym_normalize(g)
for f in (1, 37, 128, 300):
    x = torch.from_numpy(features(n, f, (f + 3) // 4 * 4, seed=f)).to(dev)
    G.gsp_spmm(gn, x, f=f)
    for r in ("mean", "max", "min"):
        G.gsp_gspmm(gn, x, r, f=f)
G.gsp_propagate(gn, torch.from_numpy(features(n, 41, 44)).to(dev), [0.1 * 0.9 ** k for k in range(4)], f=41)
H, D = 8, 16
z = torch.from_numpy(uniform((n, H * D), seed=1)).to(dev)
el, er = G.gsp_attn_project(z, torch.from_numpy(uniform(H * D, 2)).to(dev), torch.from_numpy(uniform(H * D, 3)).to(dev), H, D)
y, a = G.gsp_gat_aggregate(g, el, er, z, H, D, alpha_out=True)
G.gsp_edge_softmax(g, a, H)
G.gsp_multihead_spmm(g, a, z, H, D)
at, perm = G.gsp_csr_transpose(g)
G.gsp_sddmm(g, z, z, heads=H)
G.gsp_edge_softmax_backward(g, a, a, H)
dz, d_el, d_er = G.gsp_gat_aggregate_backward(g, at, perm, el, er, z, y, H, D)
G.gsp_attn_project_backward(z, torch.from_numpy(uniform(H * D, 2)).to(dev), torch.from_numpy(uniform(H * D, 3)).to(dev),
                            d_el, d_er, dz, H, D)
b, bd = G.gsp_partition_rows(gn, 3)
sl = G.gsp_csr_slice(gn, b, 1, max(b[i + 1] - b[i] for i in range(3)))
xin = torch.from_numpy(features(n, 50, 52)).to(dev)[:, :50]
gcn_inference(gn, xin, GCNParams.init(50, 32, 7, dev))
gat_inference(g, xin, GATParams.init(50, 32, 4, 7, dev))
# tensor-core dense step (3xTF32 tcgen05, incl. a ragged row tail and two N tiles) and fp16-storage SpMM
for (rows, fi, fo) in ((300, 37, 41), (129, 64, 300), (300, 400, 64)):  # 400: CTA pairs sharing W (3 tiles + pad)
    xl = torch.from_numpy(features(rows, fi, (fi + 3) // 4 * 4, seed=5)).to(dev)[:, :fi]
    G.gsp_linear(xl, torch.from_numpy(uniform((fi, fo), seed=6)).to(dev))
for f in (5, 128, 300):
    xh = torch.from_numpy(features(n, f, (f + 3) // 4 * 4, seed=f)).to(dev).half()
    G.gsp_spmm_f16(gn, xh, f=f)
G.gsp_gat_aggregate(g, el, er, z, H, D, single_launch=True)
# round 2: single-head / 2-head softmax with long rows (partial merge path), validate mode,
# normalisation without deg_out, the 128-byte feature layout
for hh in (1, 2, 16):
    G.gsp_edge_softmax(g, torch.from_numpy(uniform((g.nnz, hh), seed=hh)).to(dev), hh)
G.gsp_set_flags(G.GSP_VALIDATE)
G.gsp_gat_aggregate(g, el, er, z, H, D)
G.gsp_set_flags(0)
G.gsp_sym_normalize(g, keep_deg=False)
xa = G.empty_features(n, 602, dev)
xa.copy_(torch.from_numpy(features(n, 602, 602, seed=9)))
G.gsp_spmm(gn, xa)
# column blocks (split + blocked SpMM, incl. an empty block)
for bnds in ([0, n // 2, n], [0, 0, n // 3, n]):
    blocks = G.gsp_csr_colblock(gn, bnds)
    G.gsp_spmm_blocked(blocks, xa)
torch.cuda.synchronize()
print("sanitize smoke ok")
