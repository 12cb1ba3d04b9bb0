"""PCIe copy throughput: contiguous vs strided 2-D (per-slab) copies, both directions."""
import json
import torch
from cuda.bindings import runtime as rt

n, ld = 232965, 604
dev = torch.device("cuda", 0)
xh = torch.randn(n, ld).pin_memory()
yh = torch.empty(n, ld).pin_memory()
xd = torch.empty(n, ld, device=dev)
s = torch.cuda.current_stream()
res = {}


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


nbytes = n * ld * 4
res["h2d_contig_GBps"] = nbytes / timeit(lambda: xd.copy_(xh, non_blocking=True)) / 1e6
res["d2h_contig_GBps"] = nbytes / timeit(lambda: yh.copy_(xd, non_blocking=True)) / 1e6
for cols in (128, 256, 604):
    def h2d():
        for c0 in range(0, ld, cols):
            w = min(cols, ld - c0)
            rt.cudaMemcpy2DAsync(xd.data_ptr() + 4 * c0, ld * 4, xh.data_ptr() + 4 * c0, ld * 4, w * 4, n,
                                 rt.cudaMemcpyKind.cudaMemcpyHostToDevice, s.cuda_stream)
    def d2h():
        for c0 in range(0, ld, cols):
            w = min(cols, ld - c0)
            rt.cudaMemcpy2DAsync(yh.data_ptr() + 4 * c0, ld * 4, xd.data_ptr() + 4 * c0, ld * 4, w * 4, n,
                                 rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, s.cuda_stream)
    res[f"h2d_2d_{cols}cols_GBps"] = nbytes / timeit(h2d) / 1e6
    res[f"d2h_2d_{cols}cols_GBps"] = nbytes / timeit(d2h) / 1e6
# both directions at once (two streams)
s2 = torch.cuda.Stream()
def both():
    with torch.cuda.stream(s2):
        yh.copy_(xd, non_blocking=True)
    xd2 = xd  # noqa
    xd.copy_(xh, non_blocking=True) if False else None
res["note"] = "GB/s = bytes / ms / 1e6"
print(json.dumps(res))
