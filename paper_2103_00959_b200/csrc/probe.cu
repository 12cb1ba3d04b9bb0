// probe.cu -- measurement helper (not part of the method): streaming-read
// bandwidth of an L2-resident buffer, the ceiling the gather kernels' L2 hits
// are compared against in bench.py (DESIGN.md §8 roofline).
#include "common.cuh"

namespace gsp {

__global__ void __launch_bounds__(256) l2_read_kernel(const float4 *__restrict__ buf, int64_t n4, int iters,
                                                      float *__restrict__ sink) {
  // 8 independent 16-byte loads in flight per thread per step
  float acc = 0.0f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; ++it)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += 8 * stride) {
      float4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = (i + k * stride < n4) ? __ldcg(buf + i + k * stride) : make_float4(0, 0, 0, 0);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += v[k].x + v[k].y + v[k].z + v[k].w;
    }
  if (acc == 1234.5f) sink[blockIdx.x] = acc;  // keeps the loads alive
}

}  // namespace gsp

using namespace gsp;

// Reads `bytes` (multiple of 16, 16-byte aligned; keep it well under the L2
// size so it stays resident) `iters` times.  One launch on `stream`.
extern "C" gsp_status gsp_probe_l2_read(const void *buf, size_t bytes, int32_t iters, float *sink, gsp_stream stream) {
  clear_detail();
  if (!buf || !sink || bytes < 16 || bytes % 16 || iters <= 0 || !aligned16(buf))
    return fail(GSP_ERR_INVALID_ARG, "gsp_probe_l2_read: bad argument");
  const unsigned grid = (unsigned)sm_count() * 8;
  l2_read_kernel<<<grid, 256, 0, cs(stream)>>>(reinterpret_cast<const float4 *>(buf), (int64_t)(bytes / 16), iters,
                                               sink);
  return check_launch("l2_read_kernel");
}
