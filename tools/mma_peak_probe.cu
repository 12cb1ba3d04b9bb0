// mma_peak_probe.cu -- tcgen05.mma issue-bound throughput per kind on one
// B200, the denominator for the NEXT-1 GEMM's roofline: one CTA per SM, one
// elected thread issues back-to-back M=128 x N x K MMAs from fixed shared-memory
// operands into a TMEM accumulator (no memory traffic), committing every 64
// MMAs and waiting on the mbarrier only to bound the queue.  TFLOP/s = 2 M N K
// x MMAs x SMs / time (CUDA events, after a warm-up launch).  Operand values
// are whatever shared memory holds: throughput does not depend on them.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_peak_probe tools/mma_peak_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      printf("CUDA %s: %s\n", #x, cudaGetErrorString(e_));                             \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {  // K-major, SWIZZLE_64B (as linear_tc.cu)
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}

// instruction descriptor: D f32; a/b format 2 = TF32 (kind::tf32), 1 = BF16 (kind::f16); M = 128
__host__ __device__ constexpr uint32_t idesc(int n, uint32_t fmt) {
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

template <bool kTF32, int N, bool kATmem = false>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, unsigned long long *cycles) {
  extern __shared__ __align__(1024) uint8_t s_raw[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t s_tmem;
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(s_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&s_tmem))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  if (threadIdx.x == 0) {
    const uint64_t a = desc_sw64(smem_u32(base)), b = desc_sw64(smem_u32(base + 16384));
    const uint32_t id = idesc(N, kTF32 ? 2u : 1u);
    const unsigned long long t0 = clock64();
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 8
      for (int j = 0; j < 64; ++j) {
        if (kATmem)  // A operand from TMEM columns [128, 136) (N = 128 accumulator in [0, 128))
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
              "r"(tmem + 128u), "l"(b), "r"(id), "r"(1u));
        else if (kTF32)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(a), "l"(b), "r"(id), "r"(1u));
        else
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(a), "l"(b), "r"(id), "r"(1u));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bar))
                   : "memory");
      uint32_t ok = 0;
      while (!ok)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(&bar)), "r"(phase)
            : "memory");
      phase ^= 1u;
    }
    if (blockIdx.x == 0) *cycles = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

template <bool kTF32, int N, bool kATmem = false>
static int run(int sms, const char *name) {
  const int iters = 2000;
  const int smem = 64 * 1024;
  CK(cudaFuncSetAttribute(mma_loop<kTF32, N, kATmem>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  unsigned long long *d_cyc;
  CK(cudaMalloc(&d_cyc, 8));
  mma_loop<kTF32, N, kATmem><<<sms, 128, smem>>>(100, d_cyc);  // warm-up
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_loop<kTF32, N, kATmem><<<sms, 128, smem>>>(iters, d_cyc);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc = 0;
  CK(cudaMemcpy(&cyc, d_cyc, 8, cudaMemcpyDeviceToHost));
  const int K = kTF32 ? 8 : 16;  // K per MMA: 32 bytes of each operand row
  const double mmas = (double)iters * 64 * sms;
  const double flops = 2.0 * 128 * N * K * mmas;
  printf("{\"kind\": \"%s\", \"M\": 128, \"N\": %d, \"K\": %d, \"sms\": %d, \"ms\": %.4f, \"TFLOPs\": %.1f, "
         "\"clk_per_mma\": %.2f, \"flop_per_clk_per_sm\": %.0f}\n",
         name, N, K, sms, ms, flops / (ms * 1e-3) / 1e12, (double)cyc / (iters * 64.0),
         2.0 * 128 * N * K / ((double)cyc / (iters * 64.0)));
  cudaFree(d_cyc);
  return 0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  if (run<true, 128>(sms, "tf32")) return 1;
  if (run<true, 256>(sms, "tf32")) return 1;
  if (run<true, 128, true>(sms, "tf32_A_from_tmem")) return 1;
  if (run<false, 128>(sms, "bf16")) return 1;
  if (run<false, 256>(sms, "bf16")) return 1;
  return 0;
}
