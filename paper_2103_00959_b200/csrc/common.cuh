// common.cuh -- shared host/device helpers of libgsp (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <atomic>

#include "../../include/gsp.h"

namespace gsp {

// ---------------------------------------------------------------- errors
void set_detail(const char *fmt, ...);
void clear_detail();
gsp_status fail(gsp_status st, const char *fmt, ...);

inline cudaStream_t cs(gsp_stream s) { return reinterpret_cast<cudaStream_t>(s); }

// Report the first launch error of the preceding kernel(s).
gsp_status check_launch(const char *what);

int sm_count();  // cached per device

constexpr int kWarp = 32;

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline bool aligned8(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 7u) == 0; }

// Byte-range overlap test for alias checks.
inline bool overlaps(const void *a, size_t abytes, const void *b, size_t bbytes) {
  uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
  return abytes && bbytes && a0 < b0 + bbytes && b0 < a0 + abytes;
}

gsp_status check_csr(const gsp_csr *a, bool need_val, const char *fn);

// Exclusive scan of L uint32 (in may equal out), build.cu; ws >= scan_ws_bytes(L)
size_t scan_ws_bytes(int64_t L);
gsp_status scan_exclusive(const uint32_t *in, uint32_t *out, int64_t L, uint8_t *ws, cudaStream_t s);

// GSP_VALIDATE mode of the calling thread (validate.cu) and the finite check
// of logit-like inputs it enables
bool validate_mode();
gsp_status check_finite(cudaStream_t s, const char *fn, int narr, const float *const *arr, const int64_t *count,
                        const char *const *name);

// Device-side helpers --------------------------------------------------------

// Warp-cooperative lower_bound: first r in [0, n) with rp[r] >= t, or n.
// Every lane of the warp must call it; all lanes get the result.
__device__ __forceinline__ int64_t warp_lower_bound(const int64_t *__restrict__ rp, int64_t n,
                                                    int64_t t) {
  const int lane = threadIdx.x & 31;
  int64_t lo = 0, hi = n;  // answer in [lo, hi]; probes stay < hi <= n
  while (hi - lo > 31) {
    const int64_t span = hi - lo;
    const int64_t p = lo + (span * (lane + 1)) / 33;  // strictly inside [lo, hi)
    const bool ge = __ldg(rp + p) >= t;
    const unsigned b = __ballot_sync(0xffffffffu, ge);
    if (b) {
      const int j = __ffs(b) - 1;
      const int64_t pj = lo + (span * (j + 1)) / 33;
      const int64_t pjm = (j == 0) ? lo : lo + (span * j) / 33 + 1;
      hi = pj;
      lo = pjm;
    } else {
      lo = lo + (span * 32) / 33 + 1;
    }
  }
  const int64_t p = lo + lane;
  const bool ge = (p < hi) ? (__ldg(rp + p) >= t) : true;
  const unsigned b = __ballot_sync(0xffffffffu, ge);
  return lo + (__ffs(b) - 1);
}

// ---- shared-memory mbarrier + 1-D TMA bulk copy (sm_90+ / sm_100a PTX) ----
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// global -> shared bulk copy (TMA engine, no registers); 16-byte aligned, size % 16 == 0
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
// The staged CSR window is read once per CTA: its L2 lines carry an
// evict_first policy so the streamed CSR does not push the gathered X slab
// out of L2 (C4 -0.7%, fp16 C4 -1.5%, profiles/r1_sweep_variants.txt);
// -DGSP_CSR_EVICT_NORMAL turns it off.
#if !defined(GSP_CSR_EVICT_NORMAL)
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
#else
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
#endif
}

}  // namespace gsp
