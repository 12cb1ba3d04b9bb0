"""e2e probe (C4, pinned host X -> Y on the host): HostSpMM (per-slab 2-D DMA
in, gsp_spmm, 2-D DMA out) against zero-copy output -- gsp_spmm writes each
Y slab straight into the mapped pinned host buffer (posted PCIe writes from
the SMs), so only the H2D copies use the DMA engines; optionally each slab's
H2D is split over two copy streams.  Median ms of 5 after 2 warm-ups; checks
the result bitwise against the device-only path."""
import ctypes
import json
import os
import sys

import numpy as np
import torch
from cuda.bindings import runtime as rt

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_00959_b200 as G  # noqa: E402
from paper_2103_00959_b200.host import HostSpMM  # noqa: E402
from synth import CONFIGS, features, graph_for  # noqa: E402

dev = torch.device("cuda", 0)
cfg = CONFIGS["C4"]
s, d = graph_for(cfg, seed=1)
g = G.gsp_sym_normalize(G.gsp_coo_to_csr(cfg.n, torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev)))
n, f = cfg.n, cfg.f
ld = G.feature_ld(f)
xh = torch.zeros((n, ld), dtype=torch.float32).pin_memory()
xh[:, :f] = torch.from_numpy(features(n, f, f, seed=2))
yh = torch.zeros((n, ld), dtype=torch.float32).pin_memory()
xd = torch.empty((n, ld), dtype=torch.float32, device=dev)
L = G.lib()
view = g.view()
yref = G.gsp_spmm(g, xh.to(dev)[:, :f], f=f).cpu()


def copy2d(dst_ptr, dpitch, src_ptr, spitch, width, rows, kind, stream):
    err, = rt.cudaMemcpy2DAsync(dst_ptr, dpitch, src_ptr, spitch, width, rows, kind, stream.cuda_stream)
    assert err == rt.cudaError_t.cudaSuccess, err


def zero_copy(split=1, slab=128):
    main = torch.cuda.current_stream()
    cols = list(range(0, f, slab)) + [f]
    ns = len(cols) - 1
    h2d = [torch.cuda.Stream() for _ in range(split)]
    loaded = [[torch.cuda.Event() for _ in range(split)] for _ in range(ns)]
    rows = [(k * n // split, (k + 1) * n // split) for k in range(split)]

    def step():
        for st in h2d:
            st.wait_stream(main)
        for si in range(ns):
            c0, c1 = cols[si], cols[si + 1]
            for k, st in enumerate(h2d):
                r0, r1 = rows[k]
                copy2d(xd.data_ptr() + (r0 * ld + c0) * 4, ld * 4, xh.data_ptr() + (r0 * ld + c0) * 4, ld * 4,
                       (c1 - c0) * 4, r1 - r0, rt.cudaMemcpyKind.cudaMemcpyHostToDevice, st)
                loaded[si][k].record(st)
        for si in range(ns):
            c0, c1 = cols[si], cols[si + 1]
            for k in range(split):
                main.wait_event(loaded[si][k])
            st = L.gsp_spmm(ctypes.byref(view), ctypes.c_void_p(xd.data_ptr() + c0 * 4), c1 - c0, ld,
                            ctypes.c_void_p(yh.data_ptr() + c0 * 4), ld, ctypes.c_void_p(main.cuda_stream))
            assert st == 0, st
    return step


def timeit(fn, reps=5, warm=2):
    ts = []
    for i in range(warm + reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= warm:
            ts.append(a.elapsed_time(b))
    return round(float(np.median(ts)), 3)


res = {}
hs = HostSpMM(g, f, ld, device=dev)
res["HostSpMM (2-D DMA in and out)"] = timeit(lambda: hs(xh, yh))
res["HostSpMM bitwise"] = bool(torch.equal(yh[:, :f], yref))
for split in (1, 2):
    for slab in (128, 256):
        yh.zero_()
        res[f"zero-copy Y, H2D split {split}, slab {slab}"] = timeit(zero_copy(split, slab))
        res[f"zero-copy Y, H2D split {split}, slab {slab} bitwise"] = bool(torch.equal(yh[:, :f], yref))
print(json.dumps(res, indent=1))
