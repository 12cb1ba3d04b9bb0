"""PCIe 2-D slab copies (128 columns of a 232,965 x 604 fp32 matrix), both
directions at once, with each direction split over 1, 2 or 4 streams (row
ranges) -- does engine concurrency recover the contiguous-copy rate?"""
import json
import torch
from cuda.bindings import runtime as rt

n, ld, cols = 232965, 604, 128
dev = torch.device("cuda", 0)
xh = torch.randn(n, ld).pin_memory()
yh = torch.empty(n, ld).pin_memory()
xd = torch.empty(n, ld, device=dev)
yd = torch.randn(n, ld, device=dev)
H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost
main = torch.cuda.current_stream()
res = {}
for k in (1, 2, 4):
    hs = [torch.cuda.Stream() for _ in range(k)]
    ds = [torch.cuda.Stream() for _ in range(k)]

    def run():
        for st in hs + ds:
            st.wait_stream(main)
        for c0 in range(0, ld, cols):
            w = min(cols, ld - c0)
            for i in range(k):
                r0, r1 = n * i // k, n * (i + 1) // k
                rt.cudaMemcpy2DAsync(xd.data_ptr() + 4 * (r0 * ld + c0), ld * 4, xh.data_ptr() + 4 * (r0 * ld + c0),
                                     ld * 4, w * 4, r1 - r0, H2D, hs[i].cuda_stream)
                rt.cudaMemcpy2DAsync(yh.data_ptr() + 4 * (r0 * ld + c0), ld * 4, yd.data_ptr() + 4 * (r0 * ld + c0),
                                     ld * 4, w * 4, r1 - r0, D2H, ds[i].cuda_stream)
        for st in hs + ds:
            main.wait_stream(st)

    run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        run()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    res[f"streams_per_dir_{k}"] = {"ms": ms, "GBps_each_dir": n * ld * 4 / ms / 1e6}
print(json.dumps(res))
