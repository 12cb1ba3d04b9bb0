"""Timeline of one row-statistics launch (tuning probe).  Needs a libgsp built
with -DGSP_STAT_TRACE=1 (GSP_LIB=variants/libgsp_trace.so): every CTA records
its start / end (globaltimer), SM id and long-row count.  Prints the launch
span, the CTA duration distribution, the CTAs resident over time and the
slowest CTAs with their row degrees, for the C3 edge softmax (logits, H = 8)
on the power-law graph and on an Erdos-Renyi graph of the same n and nnz."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_00959_b200 as G  # noqa: E402
from synth import CONFIGS, erdos_renyi, graph_for, uniform  # noqa: E402

dev = torch.device("cuda", 0)
L = G.lib()
KMAX = 1 << 16
RPW = int(os.environ.get("RPW", "16"))
WARPS = int(os.environ.get("WARPS", "8"))


def trace(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    L.gsp_debug_stat_trace_reset()
    fn()
    torch.cuda.synchronize()
    buf = np.zeros((4, KMAX), dtype=np.uint64)
    L.gsp_debug_stat_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
    return buf


def report(name, g, buf, ncta):
    st, en, sm, nl = (buf[i, :ncta].astype(np.int64) for i in range(4))  # nl: 1 for a long-row CTA
    t0 = st.min()
    st, en = (st - t0) / 1e3, (en - t0) / 1e3  # us
    dur = en - st
    rp = g.row_ptr.cpu().numpy()
    deg = np.diff(rp)
    kr = RPW * WARPS
    nlong = int(nl.sum())
    lr = int(os.environ.get("LONG_SLICE", "128"))
    span = lambda i: slice(i * lr, (i + 1) * lr) if i < nlong else slice((i - nlong) * kr, (i - nlong + 1) * kr)
    cta_max = np.array([deg[span(i)].max(initial=0) for i in range(ncta)])
    cta_nnz = np.array([deg[span(i)].sum() for i in range(ncta)])
    bins = np.arange(0, en.max() + 1, 1.0)
    active = [int(((st <= b) & (en > b)).sum()) for b in bins]
    out = {"graph": name, "ctas": int(ncta), "span_us": round(float(en.max()), 2),
           "dur_us p50/p90/p99/max": [round(float(np.percentile(dur, q)), 2) for q in (50, 90, 99, 100)],
           "start_us p50/max": [round(float(np.median(st)), 2), round(float(st.max()), 2)],
           "active_ctas_per_us (every 4th)": active[::4],
           "slowest": [{"cta": int(i), "dur_us": round(float(dur[i]), 2), "start": round(float(st[i]), 2),
                        "long_cta": int(nl[i]), "max_deg": int(cta_max[i]), "nnz": int(cta_nnz[i])}
                       for i in np.argsort(-dur)[:8]],
           "corr(dur, max_deg)": round(float(np.corrcoef(dur, cta_max)[0, 1]), 3),
           "corr(dur, nnz)": round(float(np.corrcoef(dur, cta_nnz)[0, 1]), 3)}
    print(json.dumps(out), flush=True)


cfg = CONFIGS["C3"]
H = 8
graphs = {"chung-lu": graph_for(cfg, seed=1)}
s, d = erdos_renyi(cfg.n, cfg.m, seed=1)
graphs["erdos-renyi"] = (s, d)
for name, (s, d) in graphs.items():
    g = G.gsp_coo_to_csr(cfg.n, torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev))
    lg = torch.from_numpy(uniform((g.nnz, H), seed=4, low=-3, high=3)).to(dev)
    al = torch.empty_like(lg)
    ncta = -(-cfg.n // int(os.environ.get("LONG_SLICE", "128"))) + (cfg.n + RPW * WARPS - 1) // (RPW * WARPS)
    buf = trace(lambda: G.gsp_edge_softmax(g, lg, H, alpha=al))
    report(name + " edge_softmax", g, buf, ncta)
    el = torch.from_numpy(uniform((cfg.n, H), seed=4, low=-3, high=3)).to(dev)
    er = torch.from_numpy(uniform((cfg.n, H), seed=5, low=-3, high=3)).to(dev)
    z = torch.from_numpy(uniform((cfg.n, H * 64), seed=3)).to(dev)
    y = G.empty_features(cfg.n, H * 64, dev)
    ws = torch.empty(G.gsp_gat_workspace(g, H), dtype=torch.uint8, device=dev)
    buf = trace(lambda: G.gsp_gat_aggregate(g, el, er, z, H, 64, 0.2, y=y, ws=ws))
    report(name + " gat_stats", g, buf, ncta)
