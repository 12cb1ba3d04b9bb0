// h2d_probe.cu -- host->device bandwidth for the e2e slab copies: a
// [n][608] fp32 pinned host matrix (C4's X, 566 MB), 128-column slabs
// (512-byte row pieces): (a) cudaMemcpy2DAsync per slab, (b) an SM-driven
// copy kernel reading the mapped host rows (zero-copy, float4 per lane, 4
// rows in flight per warp), (c) one contiguous cudaMemcpyAsync of the whole
// matrix; and the same for device->host.  GB/s of payload.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o h2d_probe tools/h2d_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

// copy rows [0, n) x cols [c0, c0 + 128) from src (ld floats) to dst (ld floats)
__global__ void __launch_bounds__(256) slab_copy(const float4 *__restrict__ src, float4 *__restrict__ dst, int64_t n,
                                                 int64_t ldv, int64_t c0v) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp * 4; r < n; r += nw * 4) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (r + u < n) v[u] = src[(r + u) * ldv + c0v + lane];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (r + u < n) dst[(r + u) * ldv + c0v + lane] = v[u];
  }
}

int main() {
  const int64_t n = 232965, ld = 608, f = 602;
  const size_t bytes = (size_t)n * ld * 4;
  float *h, *d;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
  CK(cudaMalloc(&d, bytes));
  for (size_t i = 0; i < (size_t)n * ld; ++i) h[i] = (float)(i % 1000);
  float *hd;
  CK(cudaHostGetDevicePointer(&hd, h, 0));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double payload = (double)n * f * 4;
  auto report = [&](const char *name, float ms, double by) { printf("{\"probe\":\"%s\",\"ms\":%.3f,\"GBps\":%.1f}\n", name, ms, by / (ms * 1e-3) / 1e9); };
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    // (a) 2-D DMA per 128-column slab
    cudaEventRecord(a);
    for (int64_t c0 = 0; c0 < f; c0 += 128) {
      const int64_t w = (f - c0 < 128 ? f - c0 : 128);
      CK(cudaMemcpy2DAsync(d + c0, ld * 4, h + c0, ld * 4, w * 4, n, cudaMemcpyHostToDevice, 0));
    }
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    if (rep) report("h2d_2d_dma_slab128", ms, payload);
    // (b) SM-driven zero-copy reads, per slab
    for (int grid : {sms * 4, sms * 8, sms * 16}) {
      cudaEventRecord(a);
      for (int64_t c0 = 0; c0 < 640; c0 += 128)
        slab_copy<<<grid, 256>>>((const float4 *)hd, (float4 *)d, n, ld / 4, c0 / 4);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b);
      char nm[64];
      snprintf(nm, sizeof nm, "h2d_zero_copy_kernel_grid%d", grid);
      if (rep) report(nm, ms, (double)n * 640 * 4);
    }
    // (c) contiguous DMA
    cudaEventRecord(a);
    CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, 0));
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    if (rep) report("h2d_contiguous_dma", ms, (double)bytes);
    // D2H: 2-D DMA per slab and SM-driven writes into mapped host memory
    cudaEventRecord(a);
    for (int64_t c0 = 0; c0 < f; c0 += 128) {
      const int64_t w = (f - c0 < 128 ? f - c0 : 128);
      CK(cudaMemcpy2DAsync(h + c0, ld * 4, d + c0, ld * 4, w * 4, n, cudaMemcpyDeviceToHost, 0));
    }
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    if (rep) report("d2h_2d_dma_slab128", ms, payload);
    cudaEventRecord(a);
    for (int64_t c0 = 0; c0 < 640; c0 += 128)
      slab_copy<<<sms * 8, 256>>>((const float4 *)d, (float4 *)hd, n, ld / 4, c0 / 4);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    if (rep) report("d2h_zero_copy_kernel", ms, (double)n * 640 * 4);
  }
  return 0;
}
