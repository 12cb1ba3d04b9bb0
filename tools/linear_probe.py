"""gsp_linear: tcgen05 3xTF32 vs cuBLAS fp32 SGEMM on the NEXT-1 layer shapes
(n x f_in -> f_out), median ms with L2 flushed; TFLOP/s counts 2 n f_in f_out
(the useful fp32 flops, not the 3 TF32 products)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_00959_b200 as G  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res = []
for name, n, f_in, f_out in [("C4-l1", 232965, 602, 128), ("C5-l1", 716847, 300, 128), ("C3-l1", 89350, 500, 128),
                             ("C4-l2", 232965, 128, 41), ("C3-gat-l1", 89350, 500, 512)]:
    ld = (f_in + 3) // 4 * 4
    x = torch.rand((n, ld), device=dev)[:, :f_in]
    w = torch.rand((f_in, f_out), device=dev)
    y = torch.empty((n, (f_out + 3) // 4 * 4), device=dev)[:, :f_out]
    row = {"shape": name, "n": n, "f_in": f_in, "f_out": f_out}
    for tc in (True, False):
        fn = lambda: G.gsp_linear(x, w, y=y, tensor_cores=tc)
        for _ in range(3):
            fn()
        ts = []
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        row["tc_ms" if tc else "cublas_ms"] = ms
        if tc:  # error vs fp64, scaled by |x||w| (the 3xTF32 bound is 2^-19 + F_in 2^-23)
            fn()
            torch.cuda.synchronize()
            xs, ws_ = x[:4096].double(), w.double()
            ref = xs @ ws_
            row["tc_err_over_scale"] = float(((y[:4096].double() - ref).abs() / (xs.abs() @ ws_.abs())).max())
        row["tc_TFLOPs" if tc else "cublas_TFLOPs"] = 2 * n * f_in * f_out / ms / 1e9
    res.append(row)
    print(json.dumps(row), flush=True)
