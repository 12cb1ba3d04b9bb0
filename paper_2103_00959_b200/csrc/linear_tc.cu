// linear_tc.cu -- NEXT-1 dense step Y = X W (Eq. gcn_layer, "H W") on
// the 5th-generation tensor cores: tcgen05.mma kind::tf32 with fp32-accurate
// 3xTF32 splitting, operands staged by TMA, accumulator in TMEM.
//
// Why 3xTF32: the layer's parity bound is the fp32 one (DESIGN.md §NEXT rows:
// (1e-5 + F_in 2^-24) cond); a single TF32 product has 2^-11 relative error.
// With x = x_hi + x_lo and w = w_hi + w_lo, x w ~= x_lo w_hi + x_hi w_lo +
// x_hi w_hi.  W is split once (w_hi = rna_tf32(w), |w_lo| <= 2^-11 |w|).  X is
// not rewritten: kind::tf32 reads the raw fp32 tile as x_hi = trunc_tf32(x)
// (its top 19 bits; test_linear_tc_low_mantissa_bits fails by 2^-10 otherwise)
// and the converter warps store only x_lo = x - trunc_tf32(x) (exact,
// |x_lo| < 2^-10 |x|).  The MMA truncates the lo parts too; with the dropped
// x_lo w_lo the error is <= (2^-20 + 2 * 2^-21) |x||w| = 2^-19 |x||w| per
// product, accumulated in fp32 in TMEM.  (-DGSP_TC_RAWHI=0: x_hi = rna_tf32(x)
// written back, 1.25 * 2^-20.)
//
// One CTA per (128-row tile of X, <= 256 output columns): one MMA per K step
// covers the CTA's whole output tile (M = 128, N, K = 8); K in tiles of 16
// (64-byte rows, SWIZZLE_64B), 2-4 stages in <= 100 KB so two CTAs share an
// SM and one's epilogue overlaps the other's main loop.  Warp roles (6 warps):
//   warp 0 (one lane): TMA producer -- X tile [128 x 16] and the pre-split
//           W^T tiles (hi, lo) [N x 16] per stage, one mbarrier per stage;
//   warp 1: TMEM allocation; one lane issues the MMAs and tcgen05.commit;
//   warps 2-5: split the X tile in place (hi) and into the lo buffer, then
//           (after the last commit) the epilogue tcgen05.ld -> global Y.
#include <cuda.h>

#include "spmm_engine.cuh"

namespace gsp {

constexpr int kTcBM = 128, kTcBK = 16;  // K tile: 16 fp32 = 64-byte rows (SWIZZLE_64B)
constexpr int kTcNT = 256;  // max output columns per CTA (wider outputs: several adjacent CTAs per row tile)
constexpr int kTcThreads = 192;
#ifndef GSP_TC_MC
#define GSP_TC_MC 1
#endif
#ifndef GSP_TC_RAWHI
#define GSP_TC_RAWHI 1
#endif


__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// W (row-major [f_in][ldw]) -> W^T split, K-major: bt[0][n][k] = hi, bt[1][n][k] = lo,
// zero beyond f_out / f_in (n < n_pad, k < k_pad)
__global__ void split_wt_kernel(const float *__restrict__ w, int64_t ldw, int f_in, int f_out, int n_pad, int k_pad,
                                float *__restrict__ bt) {
  const int64_t total = (int64_t)n_pad * k_pad;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(i / k_pad), k = (int)(i % k_pad);
    const float v = (n < f_out && k < f_in) ? w[(int64_t)k * ldw + n] : 0.0f;
    const float hi = tf32_rna(v);
    bt[i] = hi;
    bt[total + i] = v - hi;
  }
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_64B (8-row x 64-byte atoms,
// atoms 512 B apart): start>>4 | LBO 1 | SBO 32 | version 1 | layout 4
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;           // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;  // stride byte offset: next 8-row group
  d |= (uint64_t)1 << 46;           // descriptor version (sm100)
  d |= (uint64_t)4 << 61;           // SWIZZLE_64B
  return d;
}

// instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int n) {
  return (1u << 4)                     // c_format = F32
         | (2u << 7) | (2u << 10)      // a_format, b_format = TF32
         | ((uint32_t)(n >> 3) << 17)  // N >> 3
         | ((uint32_t)(kTcBM >> 4) << 24);  // M >> 4
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *tm, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}

// A operand from TMEM (lane = row of the 128-row tile, column = K element)
__device__ __forceinline__ void mma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// TMA 2-D tile load multicast to the CTAs of ctamask (same smem offset and
// mbarrier offset in each)
__device__ __forceinline__ void tma_load_2d_mc(void *dst, const CUtensorMap *tm, int c0, int c1, uint64_t *bar,
                                               uint16_t ctamask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(ctamask)
      : "memory");
}

// MMA completion arrives on the mbarrier at this offset in every CTA of ctamask
__device__ __forceinline__ void mma_commit_mc(uint64_t *bar, uint16_t ctamask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(ctamask)
      : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

struct TcParams {
  float *y;
  int64_t n, ldy;
  int f_out, n_pad, nt, kt_count, stages;  // nt: output columns per CTA (n_pad / nt CTAs per row tile)
  uint32_t tmem_cols;
};

// kAT (outputs of <= 128 columns): x_hi / x_lo go to TMEM (the MMA's A
// operand from TMEM; accumulator + 4 A stages = 256 columns, so two CTAs
// still share an SM) and X's shared-memory slot is read once by the
// converters instead of read + rewritten and then read by three MMAs
// kMC = 2 (kAT only): CTA pairs (a cluster of two adjacent 128-row tiles)
// share the W tiles -- CTA r loads W_hi (r = 0) or W_lo (r = 1) and the TMA
// engine multicasts it into both CTAs, halving W's L2 traffic; a stage is
// refilled only after both CTAs' MMAs released it (commits multicast to both).
template <bool kAT, int kMC = 1>
__global__ void __launch_bounds__(kTcThreads, 2) linear_tc_kernel(const __grid_constant__ CUtensorMap tm_x,
                                                                 const __grid_constant__ CUtensorMap tm_b,
                                                                 const TcParams p) {
  extern __shared__ __align__(1024) uint8_t s_raw[];
  __shared__ __align__(8) uint64_t s_full[4], s_split[4], s_empty[4], s_done;
  __shared__ uint32_t s_tmem;
  // 1024-byte aligned stage buffers: A_hi [128x16], A_lo [128x16], B_hi [Nx16], B_lo [Nx16] fp32
  // (kAT: X [128x16] only -- x_hi / x_lo go to TMEM -- then B_hi, B_lo)
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(s_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t a_bytes = kTcBM * kTcBK * 4, b_bytes = (uint32_t)p.nt * kTcBK * 4;
  // 1-D grid: the CTAs of one 128-row tile (one per output-column tile) are
  // adjacent, so the X tile they all read comes from HBM once (C3 GAT layer 1
  // 0.242 -> 0.232 ms, C5 layer 1 0.384 -> 0.366)
  const int ntiles = p.n_pad / p.nt;
  const int n0 = (int)(blockIdx.x % ntiles) * p.nt;  // first output column of this CTA
  constexpr uint32_t kAParts = kAT ? 1 : 2;
  const uint32_t stage_bytes = kAParts * a_bytes + 2 * b_bytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = (int64_t)(blockIdx.x / ntiles) * kTcBM;
  // a CTA pair's padding CTA (grid rounded up to even) loads the last real
  // tile and stores nothing (its rows are >= n)
  const int64_t m0_ld = m0 < p.n ? m0 : ((p.n - 1) / kTcBM) * kTcBM;
  const int S = p.stages, KT = p.kt_count;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_split[s], 128);
      mbar_init(&s_empty[s], kMC);
    }
    mbar_init(&s_done, 1);
    fence_mbar_init();
  }
  if constexpr (kMC > 1) {  // the peer's barriers must be initialised before anything is multicast to it
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    cluster_sync_all();
  }
  const uint32_t crank = kMC > 1 ? cluster_ctarank() : 0u;
  constexpr uint16_t kMask = (uint16_t)((1u << kMC) - 1u);
  if (warp == 1) {  // TMEM accumulator: 128 lanes x tmem_cols fp32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;

  if (warp == 0) {
    if (lane == 0) {  // producer
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % S;
        if (kt >= S) mbar_wait(&s_empty[s], (uint32_t)((kt / S - 1) & 1));
        uint8_t *st = base + (size_t)s * stage_bytes;
        mbar_arrive_expect_tx(&s_full[s], a_bytes + 2 * b_bytes);
        tma_load_2d(st, &tm_x, kt * kTcBK, (int)m0_ld, &s_full[s]);
        if constexpr (kMC > 1) {  // this CTA's W part (hi or lo) into both CTAs of the pair
          tma_load_2d_mc(st + kAParts * a_bytes + crank * b_bytes, &tm_b, kt * kTcBK, (int)crank * p.n_pad + n0,
                         &s_full[s], kMask);
        } else {
          tma_load_2d(st + kAParts * a_bytes, &tm_b, kt * kTcBK, n0, &s_full[s]);
          tma_load_2d(st + kAParts * a_bytes + b_bytes, &tm_b, kt * kTcBK, p.n_pad + n0, &s_full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      const uint32_t idesc = umma_idesc_tf32(p.nt);
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % S;
        mbar_wait(&s_split[s], (uint32_t)((kt / S) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t st = smem_u32(base + (size_t)s * stage_bytes);
        const uint64_t bhi = umma_desc_sw64(st + kAParts * a_bytes), blo = umma_desc_sw64(st + kAParts * a_bytes + b_bytes);
        if constexpr (kAT) {
        const uint32_t a_t = tmem + (uint32_t)(p.nt + s * 2 * kTcBK);  // x_hi columns, then x_lo
#pragma unroll
        for (int kk = 0; kk < kTcBK / 8; ++kk) {  // K = 8 tf32 per MMA: 8 TMEM columns of A, 32 bytes of B
          const uint64_t o = (uint64_t)(kk * 2);
          const uint32_t acc = (kt > 0 || kk > 0) ? 1u : 0u;
          mma_tf32_ta(tmem, a_t + kTcBK + kk * 8, bhi + o, idesc, acc);  // small terms first
          mma_tf32_ta(tmem, a_t + kk * 8, blo + o, idesc, 1u);
          mma_tf32_ta(tmem, a_t + kk * 8, bhi + o, idesc, 1u);
        }
        } else {
        const uint64_t ahi = umma_desc_sw64(st), alo = umma_desc_sw64(st + a_bytes);
#pragma unroll
        for (int kk = 0; kk < kTcBK / 8; ++kk) {  // K = 8 tf32 (32 bytes) per MMA: advance start by 2 (x16 B) inside the atom
          const uint64_t o = (uint64_t)(kk * 2);
          const uint32_t acc = (kt > 0 || kk > 0) ? 1u : 0u;
          mma_tf32(tmem, alo + o, bhi + o, idesc, acc);  // small terms first
          mma_tf32(tmem, ahi + o, blo + o, idesc, 1u);
          mma_tf32(tmem, ahi + o, bhi + o, idesc, 1u);
        }
        }
        if constexpr (kMC > 1) mma_commit_mc(&s_empty[s], kMask);  // both CTAs' W slots
        else mma_commit(&s_empty[s]);  // stage reusable once these MMAs have read it
      }
      mma_commit(&s_done);
    }
  } else {
    // warps 2-5: split X tiles, then the epilogue
    const int t = threadIdx.x - 64;  // 0..127
    if constexpr (kAT) {
    // thread = one row of the tile, in this warp's TMEM lane quadrant: read the
    // row's 16 values from the SWIZZLE_64B tile (16-byte chunk c of row r sits
    // at chunk c ^ ((r >> 1) & 3)), store x (the MMA reads it as trunc_tf32(x))
    // and x - trunc_tf32(x) into the stage's TMEM columns
    (void)t;
    const int arow = (warp & 3) * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % S;
      mbar_wait(&s_full[s], (uint32_t)((kt / S) & 1));
      const uint8_t *xt = base + (size_t)s * stage_bytes + (size_t)arow * 64;
      uint32_t xh[16], xl[16];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float4 v = *reinterpret_cast<const float4 *>(xt + ((c ^ ((arow >> 1) & 3)) << 4));
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          xh[4 * c + i] = __float_as_uint(vv[i]);
          xl[4 * c + i] = __float_as_uint(vv[i] - __uint_as_float(__float_as_uint(vv[i]) & 0xffffe000u));
        }
      }
      const uint32_t acol = (uint32_t)(p.nt + s * 2 * kTcBK);
      tmem_st16(lane_base + acol, xh);
      tmem_st16(lane_base + acol + kTcBK, xl);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&s_split[s]);
    }
    } else {
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % S;
      mbar_wait(&s_full[s], (uint32_t)((kt / S) & 1));
      float4 *hi = reinterpret_cast<float4 *>(base + (size_t)s * stage_bytes);
      float4 *lo = reinterpret_cast<float4 *>(base + (size_t)s * stage_bytes + a_bytes);
#pragma unroll
      for (int i = 0; i < (int)(kTcBM * kTcBK / 4 / 128); ++i) {  // elementwise: same swizzled offset in hi and lo
        const int q = t + 128 * i;
        const float4 v = hi[q];
#if GSP_TC_RAWHI
        // the MMA reads the raw fp32 X as x_hi (kind::tf32 uses its top 19
        // bits: truncation, tested); lo = x - trunc_tf32(x) is exact
        float4 l;
        l.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xffffe000u);
        l.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xffffe000u);
        l.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xffffe000u);
        l.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xffffe000u);
        lo[q] = l;
#else
        float4 h, l;
        h.x = tf32_rna(v.x); l.x = v.x - h.x;
        h.y = tf32_rna(v.y); l.y = v.y - h.y;
        h.z = tf32_rna(v.z); l.z = v.z - h.z;
        h.w = tf32_rna(v.w); l.w = v.w - h.w;
        hi[q] = h;
        lo[q] = l;
#endif
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core (async) proxy
      mbar_arrive(&s_split[s]);
    }
    }
    // epilogue: warp w reads TMEM lanes 32*(w%4) .. +31 (rows of the tile)
    mbar_wait(&s_done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int quad = warp & 3;
    const int64_t row = m0 + quad * 32 + lane;
    for (int c0 = 0; c0 < p.nt; c0 += 16) {
      uint32_t r[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (row < p.n) {
        float *yr = p.y + row * p.ldy + n0 + c0;
        const int nv = min(16, p.f_out - n0 - c0);
        if (nv == 16 && (p.ldy % 4) == 0 && (reinterpret_cast<uintptr_t>(p.y) & 15u) == 0) {  // n0 % 16 == 0
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            *reinterpret_cast<float4 *>(yr + j) = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                              __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < nv) yr[j] = __uint_as_float(r[j]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  // no CTA of a pair exits while its peer may still multicast into it or
  // arrive on its barriers (every MMA of both has completed past this point)
  if constexpr (kMC > 1) cluster_sync_all();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols) : "memory");
  }
}

// ------------------------------------------------------------------ host
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static const EncodeTiledFn fn = []() -> EncodeTiledFn {  // thread-safe one-time lookup
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiledFn>(p);
    return nullptr;
  }();
  return fn;
}

static bool make_map_2d(CUtensorMap *m, const float *ptr, int64_t inner, int64_t rows, int64_t ld, int box_inner,
                        int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// output tiling: ntiles CTAs along N of nt columns (16-multiples <= 256), n_pad = ntiles * nt
static void tc_dims(int64_t f_out, int *nt, int *ntiles, int *n_pad) {
  const int n16 = (int)((f_out + 15) / 16);
  *ntiles = (n16 * 16 + kTcNT - 1) / kTcNT;
  *nt = ((n16 + *ntiles - 1) / *ntiles) * 16;
  *n_pad = *ntiles * *nt;
}

size_t linear_tc_ws_bytes(int64_t f_in, int64_t f_out) {
  int nt, ntiles, n_pad;
  tc_dims(std::max<int64_t>(f_out, 1), &nt, &ntiles, &n_pad);
  const int64_t k_pad = (f_in + kTcBK - 1) / kTcBK * kTcBK;
  return (size_t)(2 * (int64_t)n_pad * k_pad * 4) + 1024;
}

// true if the tensor-core path takes this GEMM (else the caller uses cuBLAS)
bool linear_tc_eligible(int64_t n, int64_t f_in, const float *x, int64_t ldx, int64_t f_out, void *ws,
                        size_t ws_bytes) {
  return ws && ws_bytes >= linear_tc_ws_bytes(f_in, f_out) && f_out >= 1 && f_out <= 4096 && f_in >= 1 &&
         ldx % 4 == 0 && aligned16(x) && n < (int64_t(1) << 31) && encode_fn() != nullptr;
}

gsp_status linear_tc(int64_t n, int64_t f_in, const float *x, int64_t ldx, const float *w, int64_t ldw,
                     int64_t f_out, float *y, int64_t ldy, void *ws, cudaStream_t s) {
  int nt, ntiles, n_pad;
  tc_dims(f_out, &nt, &ntiles, &n_pad);
  const int k_pad = (int)((f_in + kTcBK - 1) / kTcBK * kTcBK);
  float *bt = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(ws) + 1023) & ~uintptr_t(1023));
  split_wt_kernel<<<(unsigned)std::min<int64_t>(ceil_div((int64_t)n_pad * k_pad, 256), 1024), 256, 0, s>>>(
      w, ldw, (int)f_in, (int)f_out, n_pad, k_pad, bt);
  gsp_status st = check_launch("split_wt");
  if (st) return st;
  CUtensorMap tx, tb;
  if (!make_map_2d(&tx, x, f_in, n, ldx, kTcBK, kTcBM) || !make_map_2d(&tb, bt, k_pad, 2 * n_pad, k_pad, kTcBK, nt))
    return fail(GSP_ERR_CUDA, "gsp_linear: cuTensorMapEncodeTiled failed");
  TcParams p;
  p.y = y;
  p.n = n;
  p.ldy = ldy;
  p.f_out = (int)f_out;
  p.n_pad = n_pad;
  p.nt = nt;
  p.kt_count = (int)((f_in + kTcBK - 1) / kTcBK);
  const bool at = nt <= 128;  // x_hi / x_lo in TMEM (see linear_tc_kernel<true>)
  const size_t stage = (size_t)(at ? 1 : 2) * kTcBM * kTcBK * 4 + (size_t)2 * nt * kTcBK * 4;
  int stages = (int)std::min<size_t>(4, (100u * 1024u) / stage);  // <= ~100 KB: 2 CTAs per SM
  p.stages = std::max(stages, 2);
  uint32_t cols = 32;
  while ((int)cols < nt + (at ? p.stages * 2 * kTcBK : 0)) cols *= 2;  // accumulator (+ A stages)
  p.tmem_cols = cols;
  const size_t smem = (size_t)p.stages * stage + 1024;
  // CTA pairs sharing W (linear_tc_kernel<true, 2>) for long K: C4 layer 1
  // (F_in 602) 0.222 -> 0.211 ms, C3 layer 1 (500) 0.091 -> 0.089; shorter K
  // measured slower (C5 layer 1, F_in 300: 0.371 -> 0.380; F_in 128: +15%)
  const bool mc = at && GSP_TC_MC && f_in >= 384;
  const int var = mc ? 2 : (at ? 1 : 0);
  static std::atomic<int> granted[3][64];  // per kernel variant and device: largest dynamic smem already granted
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || granted[var][dev].load(std::memory_order_relaxed) < (int)smem) {
    const cudaError_t e =
        mc ? cudaFuncSetAttribute(linear_tc_kernel<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
        : at ? cudaFuncSetAttribute(linear_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
             : cudaFuncSetAttribute(linear_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return check_launch("cudaFuncSetAttribute(linear_tc_kernel)");
    if (dev >= 0 && dev < 64) granted[var][dev].store((int)smem, std::memory_order_relaxed);
  }
  if (mc) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((ceil_div(n, kTcBM) + 1) / 2 * 2));
    cfg.blockDim = dim3(kTcThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, linear_tc_kernel<true, 2>, tx, tb, p) != cudaSuccess)
      return check_launch("cudaLaunchKernelEx(linear_tc_kernel<true, 2>)");
    return check_launch("linear_tc_kernel<true, 2>");
  }
  const dim3 grid((unsigned)(ceil_div(n, kTcBM) * ntiles));
  if (at) linear_tc_kernel<true><<<grid, kTcThreads, smem, s>>>(tx, tb, p);
  else linear_tc_kernel<false><<<grid, kTcThreads, smem, s>>>(tx, tb, p);
  return check_launch("linear_tc_kernel");
}

}  // namespace gsp
