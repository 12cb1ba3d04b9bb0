// probe_gather4.cu -- standalone probe of TMA row gathers on sm_100a
// (cp.async.bulk.tensor.2d ... tile::gather4): (1) which box shape the
// tensor map needs and what lands in shared memory, (2) random 512-byte
// row-gather throughput of a per-warp TMA ring vs register LDG.128 chunks,
// with X L2-resident and X >> L2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o probe_gather4 tools/probe_gather4.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiled encode() {
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return (EncodeTiled)fn;
}
static CUtensorMap make_map(float *x, int64_t rows, int64_t cols, int64_t ld, int bw, int bh, int l2promo = 2) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        (CUtensorMapL2promotion)l2promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode(box %d x %d) failed: %d\n", bw, bh, (int)r);
  return m;
}

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
  }
}
__device__ __forceinline__ void g4(void *dst, const CUtensorMap *tm, int c0, int r0, int r1, int r2, int r3, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      ::"r"(su32(dst)), "l"(tm), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(bar)) : "memory");
}

// (1) shape test: gather rows idx[0..3] at column c0 into smem and dump it
__global__ void shape_test(const __grid_constant__ CUtensorMap tm, const int *idx, int c0, int bytes, float *out) {
  __shared__ __align__(128) float buf[4 * 256];
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) buf[i] = -1.0f;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_expect(&bar, bytes);
    g4(buf, &tm, c0, idx[0], idx[1], idx[2], idx[3], &bar);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) out[i] = buf[i];
}

// (2a) TMA ring: each warp streams its share of random rows (4 per gather4,
// 8 per stage), NS stages in flight; lanes sum float4 of each row from smem.
template <int NS>
__global__ void __launch_bounds__(256) ring_kernel(const __grid_constant__ CUtensorMap tm, const int *__restrict__ idx,
                                                   int64_t per_warp, float *sink) {
  extern __shared__ __align__(128) uint8_t dyn[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  float *ring = reinterpret_cast<float *>(dyn) + (size_t)warp * NS * 8 * 128;
  __shared__ __align__(8) uint64_t bars[8][NS];
  if (lane == 0)
    for (int s = 0; s < NS; ++s) mbar_init(&bars[warp][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t gw = (int64_t)blockIdx.x * nw + warp;
  const int *my = idx + gw * per_warp;
  const int64_t nst = per_warp / 8;
  auto issue = [&](int64_t st) {
    const int s = (int)(st % NS);
    float *dst = ring + s * 8 * 128;
    const int *q = my + st * 8;
    mbar_expect(&bars[warp][s], 8 * 512);
    g4(dst, &tm, 0, q[0], q[1], q[2], q[3], &bars[warp][s]);
    g4(dst + 4 * 128, &tm, 0, q[4], q[5], q[6], q[7], &bars[warp][s]);
  };
  if (lane == 0)
    for (int64_t st = 0; st < NS - 1 && st < nst; ++st) issue(st);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t st = 0; st < nst; ++st) {
    if (lane == 0 && st + NS - 1 < nst) issue(st + NS - 1);
    const int s = (int)(st % NS);
    mbar_wait(&bars[warp][s], (uint32_t)((st / NS) & 1));
    const float4 *b = reinterpret_cast<const float4 *>(ring + s * 8 * 128);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float4 v = b[e * 32 + lane];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    __syncwarp();  // slot s is reissued next iteration+NS-1 by lane 0 after everyone read it
  }
  sink[(blockIdx.x * blockDim.x + threadIdx.x) & 4095] = acc.x + acc.y + acc.z + acc.w;
}

// (2b) register LDG.128: U rows in flight per lane (the current engine's pattern)
template <int U>
__global__ void __launch_bounds__(256, 4) ldg_kernel(const float *__restrict__ x, int64_t ld, const int *__restrict__ idx,
                                                     int64_t per_warp, float *sink) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * nw + warp;
  const int *my = idx + gw * per_warp;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t e = 0; e < per_warp; e += U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(reinterpret_cast<const float4 *>(x + (int64_t)my[e + u] * ld) + lane);
#pragma unroll
    for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
  }
  sink[(blockIdx.x * blockDim.x + threadIdx.x) & 4095] = acc.x + acc.y + acc.z + acc.w;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  // ---- (1) shape ----
  const int64_t R = 1000, C = 300, LD = 304;
  std::vector<float> hx(R * LD);
  for (int64_t r = 0; r < R; ++r)
    for (int64_t c = 0; c < LD; ++c) hx[r * LD + c] = c < C ? (float)(r * 1000 + c) : -7.0f;
  float *dx, *dout;
  int *didx;
  CK(cudaMalloc(&dx, hx.size() * 4));
  CK(cudaMalloc(&dout, 4 * 256 * 4));
  CK(cudaMalloc(&didx, 16));
  CK(cudaMemcpy(dx, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice));
  int hidx[4] = {5, 999, 17, 1000};  // 1000 is out of range -> zero fill?
  CK(cudaMemcpy(didx, hidx, 16, cudaMemcpyHostToDevice));
  for (int bh : {1}) {  // box height 4 traps (illegal instruction): gather4 takes box {w, 1}
    for (int c0 : {0, 256}) {
      CUtensorMap tm = make_map(dx, R, C, LD, 128, bh);
      CK(cudaMemset(dout, 0, 4 * 256 * 4));
      shape_test<<<1, 128>>>(tm, didx, c0, 4 * 128 * 4, dout);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<float> o(4 * 256);
      if (e == cudaSuccess) CK(cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost));
      int bad = 0;
      for (int k = 0; k < 4 && e == cudaSuccess; ++k)
        for (int c = 0; c < 128; ++c) {
          const int64_t col = c0 + c;
          const float want = (hidx[k] < R && col < C) ? (float)(hidx[k] * 1000 + col) : 0.0f;
          if (o[k * 128 + c] != want) ++bad;
        }
      printf("{\"probe\":\"shape\",\"box_h\":%d,\"c0\":%d,\"status\":\"%s\",\"mismatches\":%d,\"row0_c0\":%g,\"row3_c0\":%g,\"after\":%g}\n",
             bh, c0, cudaGetErrorString(e), bad, o[0], o[3 * 128], o[4 * 128]);
      if (e != cudaSuccess) return 1;
    }
  }
  // ---- (2) throughput ----
  float *sink;
  CK(cudaMalloc(&sink, 4096 * 4));
  for (int64_t rows : {32768LL, 1100000LL}) {  // 16 MB (L2-resident) and 563 MB (>> L2) at ld 128
    const int64_t ld = 128;
    float *x;
    CK(cudaMalloc(&x, rows * ld * 4));
    CK(cudaMemset(x, 0, rows * ld * 4));
    const int64_t per_warp = 4096;
    const int64_t warps = (int64_t)sms * 16 * 4;
    std::vector<int> hi(warps * per_warp);
    std::mt19937_64 rng(1);
    for (auto &v : hi) v = (int)(rng() % rows);
    int *di;
    CK(cudaMalloc(&di, hi.size() * 4));
    CK(cudaMemcpy(di, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice));
    CUtensorMap tm = make_map(x, rows, ld, ld, 128, 1);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto launch) {
      launch();
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a);
      for (int i = 0; i < 5; ++i) launch();
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      return ms / 5;
    };
    const double bytes = (double)warps * per_warp * 512;
    {
      auto ms = timeit([&] { ldg_kernel<8><<<warps / 8, 256>>>(x, ld, di, per_warp, sink); });
      printf("{\"probe\":\"ldg\",\"U\":8,\"x_MB\":%.0f,\"GBps\":%.1f}\n", rows * ld * 4 / 1e6, bytes / ms / 1e6);
    }
#define RING(NS, WPC)                                                                                     \
    {                                                                                                     \
      const size_t sm = (size_t)WPC * NS * 8 * 512;                                                        \
      CK(cudaFuncSetAttribute(ring_kernel<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));     \
      auto ms = timeit([&] { ring_kernel<NS><<<warps / WPC, WPC * 32, sm>>>(tm, di, per_warp, sink); });   \
      printf("{\"probe\":\"tma_ring\",\"NS\":%d,\"warps_per_cta\":%d,\"smem_KB\":%zu,\"x_MB\":%.0f,\"GBps\":%.1f}\n", NS, WPC, \
             sm / 1024, rows * ld * 4 / 1e6, bytes / ms / 1e6);                                             \
    }
    RING(2, 8) RING(3, 8) RING(4, 8) RING(6, 4) RING(4, 4) RING(8, 2) RING(12, 2)
    CK(cudaGetLastError());
    cudaFree(x);
    cudaFree(di);
  }
  return 0;
}
