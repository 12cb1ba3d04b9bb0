// l2cap_probe.cu -- effective L2 capacity for the SpMM gather pattern:
// random 512-byte row gathers (a warp reads one row per LDG.128, 8 rows in
// flight per lane, 8 warps x 4 CTAs per SM) from an X of S MB, after one
// warm-up pass; GB/s of gathered bytes vs S.  A knee near 126 MB means the
// whole L2 holds X; a knee near half of it means lines are kept per die.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2cap_probe tools/l2cap_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

template <int MINB, int U>
__global__ void __launch_bounds__(256, MINB) gather(const float4 *__restrict__ x, const uint32_t *__restrict__ idx,
                                                 int64_t nidx, float *out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t base = warp * U; base < nidx; base += nw * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t r = idx[base + u];
      v[u] = __ldg(x + (int64_t)r * 32 + lane);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc.x += v[u].x;
      acc.y += v[u].y;
      acc.z += v[u].z;
      acc.w += v[u].w;
    }
  }
  if (acc.x == 12345.f) out[0] = acc.y + acc.z + acc.w;
}

int main() {
  const int64_t nidx = 1 << 24;  // 16M gathers x 512 B = 8.6 GB per pass
  uint32_t *d_idx;
  float4 *d_x;
  float *d_out;
  const int64_t max_mb = 512;
  CK(cudaMalloc(&d_x, max_mb << 20));
  CK(cudaMemset(d_x, 0, max_mb << 20));
  CK(cudaMalloc(&d_idx, nidx * 4));
  CK(cudaMalloc(&d_out, 4));
  std::vector<uint32_t> h(nidx);
  std::mt19937_64 rng(1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int sizes[] = {64, 96, 119, 128, 160, 256};
  auto run = [&](auto kern, int ctas, const char *name, int mb) {
    kern<<<sms * ctas, 256>>>(d_x, d_idx, nidx, d_out);  // warm-up pass
    cudaDeviceSynchronize();
    float best = 1e9f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      kern<<<sms * ctas, 256>>>(d_x, d_idx, nidx, d_out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("{\"probe\":\"l2cap\",\"kernel\":\"%s\",\"x_MB\":%d,\"ms\":%.3f,\"GBps\":%.1f}\n", name, mb, best,
           nidx * 512.0 / (best * 1e-3) / 1e9);
  };
  for (int mb : sizes) {
    const uint64_t rows = ((uint64_t)mb << 20) / 512;
    for (int64_t i = 0; i < nidx; ++i) h[i] = (uint32_t)(rng() % rows);
    CK(cudaMemcpy(d_idx, h.data(), nidx * 4, cudaMemcpyHostToDevice));
    run(gather<4, 8>, 4, "4cta_u8", mb);
    run(gather<6, 8>, 6, "6cta_u8", mb);
    run(gather<8, 8>, 8, "8cta_u8", mb);
    run(gather<4, 12>, 4, "4cta_u12", mb);
    run(gather<4, 16>, 4, "4cta_u16", mb);
    run(gather<2, 16>, 2, "2cta_u16", mb);
  }
  return 0;
}
