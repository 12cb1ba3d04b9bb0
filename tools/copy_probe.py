"""PCIe copy throughput: contiguous vs strided 2-D (per-slab) copies, each
direction alone and both directions at once (two streams, full duplex)."""
import json
import torch
from cuda.bindings import runtime as rt

n, ld = 232965, 604
dev = torch.device("cuda", 0)
xh = torch.randn(n, ld).pin_memory()
yh = torch.empty(n, ld).pin_memory()
xd = torch.empty(n, ld, device=dev)
yd = torch.randn(n, ld, device=dev)
s = torch.cuda.current_stream()
s2 = torch.cuda.Stream()
res = {}
H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost


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


def slabs(dst, src, kind, cols, stream):
    for c0 in range(0, ld, cols):
        w = min(cols, ld - c0)
        rt.cudaMemcpy2DAsync(dst.data_ptr() + 4 * c0, ld * 4, src.data_ptr() + 4 * c0, ld * 4, w * 4, n, kind,
                             stream.cuda_stream)


nbytes = n * ld * 4
res["h2d_contig_GBps"] = nbytes / timeit(lambda: xd.copy_(xh, non_blocking=True)) / 1e6
res["d2h_contig_GBps"] = nbytes / timeit(lambda: yh.copy_(yd, non_blocking=True)) / 1e6


def both_contig():
    s2.wait_stream(s)
    with torch.cuda.stream(s2):
        yh.copy_(yd, non_blocking=True)
    xd.copy_(xh, non_blocking=True)
    s.wait_stream(s2)


res["both_contig_GBps_each_dir"] = nbytes / timeit(both_contig) / 1e6
for cols in (32, 64, 128, 256):
    res[f"h2d_2d_{cols}cols_GBps"] = nbytes / timeit(lambda: slabs(xd, xh, H2D, cols, s)) / 1e6
    res[f"d2h_2d_{cols}cols_GBps"] = nbytes / timeit(lambda: slabs(yh, yd, D2H, cols, s)) / 1e6

    def both():
        s2.wait_stream(s)
        slabs(yh, yd, D2H, cols, s2)
        slabs(xd, xh, H2D, cols, s)
        s.wait_stream(s2)

    res[f"both_2d_{cols}cols_GBps_each_dir"] = nbytes / timeit(both) / 1e6
res["note"] = "GB/s = bytes / ms / 1e6; n=232965 rows, ld=604 fp32"
print(json.dumps(res))
