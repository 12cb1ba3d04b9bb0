// gat.cu -- GAT path: attention projection (a4), edge softmax (a6) and the
// fused score -> softmax -> multi-head SpMM aggregate (a5+a6+a7).
// PAPER.md P:253 (GAT), P:648-649 (multi-head SpMM), P:653-656 (edge-wise
// softmax with warp-level max / sum reductions); readings A9-A14.
#include "spmm_engine.cuh"

namespace gsp {

// ------------------------------------------------------------------------
// Row statistics: m[u,h] = max_e s[e,h] (fp64) and 1 / sum_e exp(s - m),
// all heads of a row at once (P:653-656 edge-wise softmax: "find the max
// value ... subtract ... exponent ... reduce ... the sum").  H (heads,
// dividing 32) is a template parameter.  Grid: one CTA of 8 warps per
// 8 * 32 / H rows; warp w owns RPW = 32 / H consecutive rows.
//  * SHORT rows (<= kTile = 1024 / H entries): staged in the warp's 4 KB
//    shared tile T[j][H] by cp.async (no registers in flight), as many
//    consecutive rows at a time as fit, and reduced one row at a time by the
//    whole warp (lane = (entry slot, head), xor tree over the slots).
//  * LONG rows: cut into tile-sized chunks; warp w takes chunks w, w+8, ...
//    and folds them into a partial (own max m_w, fp64 sum of exp(s - m_w));
//    the last warp to arrive merges the 8 partials in warp order (no CTA
//    barrier per long row; see row_stats_warp).
// Every order depends on the row alone (deterministic, partition-invariant).
// ------------------------------------------------------------------------
// kScores: s from el/er (GAT) or s = logits (edge softmax).
// kApply : write alpha = exp(s - m) / sum (standalone edge softmax; logits
//          may alias alpha) instead of storing the statistics.
#ifndef GSP_STAT_WARPS
#define GSP_STAT_WARPS 8
#endif
#ifndef GSP_STAT_MINB
#define GSP_STAT_MINB 4
#endif
constexpr int kStatWarps = GSP_STAT_WARPS;  // warps per CTA
constexpr int kStatTileFloats = 1024;  // per warp: kTile = 1024 / H entries x H heads (4 KB)

constexpr double kLog2e = 1.4426950408889634074;  // log2(e)
// 2^a, hardware approximation (max error 2 ulp; subnormal results kept)
__device__ __forceinline__ float ex2_approx(float a) {
  float r;
  asm("ex2.approx.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}

template <bool kScores>
__device__ __forceinline__ double stat_score(float t, double el_u, double slope) {
  if (kScores) {
    const double x = el_u + (double)t;
    return x >= 0.0 ? x : slope * x;
  }
  return (double)t;
}

// exp(s - m) for a stored value t (er of the column, or the logit), as the
// short rows form it (see stat_short_rows): 2^((s - m) log2 e)
template <bool kScores>
__device__ __forceinline__ float stat_exp(float t, double el_u, double slope_l2e, double m) {
  float a;
  if (kScores) {
    const double x = el_u + (double)t;
    a = (float)fma(x, x >= 0.0 ? kLog2e : slope_l2e, -(m * kLog2e));
  } else {
    a = (t - (float)m) * (float)kLog2e;
  }
  return ex2_approx(a);
}

// global -> shared asynchronous copies (LDGSTS): the data never passes through
// registers, so a lane keeps many entries in flight at no register cost
template <int B>
__device__ __forceinline__ void cp_async(void *dst, const void *src) {
  if constexpr (B == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(B) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// entries [e0, e0 + cnt) of the CSR -> T[j][H] (er rows of their columns, or
// logits rows) by cp.async, issued only (stat_load waits for them); the
// caller's __syncwarp after the wait publishes T
template <int H, bool kScores>
__device__ __forceinline__ void stat_load_async(float *T, int64_t e0, int cnt, const int32_t *__restrict__ col,
                                                const float *__restrict__ er, const float *logits, int lane) {
  if (kScores) {
    constexpr int kV = H >= 4 ? 4 : H;  // floats per copy (er rows are 4 / 8 / 16-byte aligned, launch_stats)
    constexpr int kU = 8;               // column indices in flight per lane
    for (int base = 0; base < cnt; base += 32 * kU) {
      int c[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int j = base + lane + 32 * u;
        c[u] = j < cnt ? __ldg(col + e0 + j) : 0;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int j = base + lane + 32 * u;
        if (j < cnt) {
#pragma unroll
          for (int q = 0; q < H; q += kV) cp_async<kV * 4>(T + j * H + q, er + (int64_t)c[u] * H + q);
        }
      }
    }
  } else {
    const float *src = logits + e0 * H;  // cnt rows of H logits are contiguous
    const int nf = cnt * H;
    int k0 = 0;
    if ((reinterpret_cast<uintptr_t>(src) & 15u) == 0) {  // T is 16-byte aligned: 16-byte copies, scalar tail
      k0 = nf & ~3;
      for (int k = 4 * lane; k < k0; k += 128) cp_async<16>(T + k, src + k);
    }
    for (int k = k0 + lane; k < nf; k += 32) cp_async<4>(T + k, src + k);
  }
}

template <int H, bool kScores>
__device__ __forceinline__ void stat_load(float *T, int64_t e0, int cnt, const int32_t *__restrict__ col,
                                          const float *__restrict__ er, const float *logits, int lane) {
  stat_load_async<H, kScores>(T, e0, cnt, col, er, logits, lane);
  cp_async_wait_all();
}

// copy alpha values staged in the warp's tile (T[j][H], entries e0 .. e0+cnt)
// to global alpha: [nnz][H] (ahs == 0: one contiguous run) or head-major
// [H][ahs] (one contiguous run per head) -- 128-byte stores either way
template <int H>
__device__ __forceinline__ void stat_store_alpha(const float *T, int64_t e0, int cnt, float *alpha, int64_t ahs,
                                                 int lane) {
  if (ahs == 0) {
    float *dst = alpha + e0 * H;
    const int nf = cnt * H;
    int k0 = 0;
    if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {  // 16-byte stores, scalar tail
      k0 = nf & ~3;
      for (int k = 4 * lane; k < k0; k += 128)
        *reinterpret_cast<float4 *>(dst + k) = *reinterpret_cast<const float4 *>(T + k);
    }
    for (int k = k0 + lane; k < nf; k += 32) dst[k] = T[k];
  } else if constexpr (H % 4 == 0) {
    // transpose through registers: lane k reads float4 k of the tile (entry
    // k / Q, heads 4 (k % Q) .. + 3; conflict-free) and writes one value into
    // each of those 4 head runs -- a store instruction covers 4 Q-entry runs
    constexpr int Q = H / 4;
    for (int k = lane; k < cnt * Q; k += 32) {
      const float4 v = reinterpret_cast<const float4 *>(T)[k];
      float *dst = alpha + (int64_t)(4 * (k % Q)) * ahs + e0 + k / Q;
      dst[0] = v.x;
      dst[ahs] = v.y;
      dst[2 * ahs] = v.z;
      dst[3 * ahs] = v.w;
    }
  } else {
#pragma unroll
    for (int h = 0; h < H; ++h)
      for (int j = lane; j < cnt; j += 32) alpha[h * ahs + e0 + j] = T[j * H + h];
  }
}

// Short rows (<= kTile entries): warp w owns rows w * RPW .. + RPW - 1 (RPW =
// 32 / H).  The rows' entries (contiguous in CSR) are staged in the warp's
// tile by cp.async, as many consecutive short rows at a time as fit, and the
// warp reduces them one row at a time: lane (part, h) takes entries part,
// part + P, ... of head h (P = 32 / H), an xor tree over the P parts
// finishes -- no lane waits on a longer row of another lane.  The row max of
// the fp64 scores is the score of the fp32 max of the stored values (LeakyReLU
// with slope >= 0 and IEEE rounding are monotone) -- exactly; slope < 0 takes
// the fp64 max of the scores.
// alpha of a batch: T holds exp(s - m) per entry and head, row_of[j] the
// batch row of entry j and inv[q * H + h] its 1 / S -- scaled on the way out
template <int H>
__device__ __forceinline__ float stat_scale(const float *T, const uint8_t *row_of, const float *inv, int f) {
  return T[f] * inv[row_of[f / H] * H + f % H];
}
template <int H>
__device__ __forceinline__ void stat_store_scaled(const float *T, const uint8_t *row_of, const float *inv, int64_t e0,
                                                  int cnt, float *alpha, int64_t ahs, int lane) {
  const int nf = cnt * H;
  constexpr int Q = H % 4 == 0 ? H / 4 : 1;  // float4s per entry (head-major transpose)
  if (ahs == 0 || H % 4 != 0) {
    // [nnz][H]: one contiguous run (head-major with H % 4 != 0: per head)
    if (ahs == 0) {
      float *dst = alpha + e0 * H;
      int k0 = 0;
      if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
        k0 = nf & ~3;
        for (int f = 4 * lane; f < k0; f += 128)
          *reinterpret_cast<float4 *>(dst + f) =
              make_float4(stat_scale<H>(T, row_of, inv, f), stat_scale<H>(T, row_of, inv, f + 1),
                          stat_scale<H>(T, row_of, inv, f + 2), stat_scale<H>(T, row_of, inv, f + 3));
      }
      for (int f = k0 + lane; f < nf; f += 32) dst[f] = stat_scale<H>(T, row_of, inv, f);
    } else {
#pragma unroll
      for (int h = 0; h < H; ++h)
        for (int j = lane; j < cnt; j += 32) alpha[h * ahs + e0 + j] = stat_scale<H>(T, row_of, inv, j * H + h);
    }
  } else {
    // head-major [H][ahs], H % 4 == 0: lane reads float4 k of the tile (entry
    // k / Q, heads 4 (k % Q) .. + 3; conflict-free) and writes one value into
    // each of those 4 head runs -- a store instruction covers 4 Q-entry runs
    for (int k = lane; k < cnt * Q; k += 32) {
      const int j = k / Q, h0 = 4 * (k % Q);
      const float4 v = reinterpret_cast<const float4 *>(T)[k];
      const float4 w = *reinterpret_cast<const float4 *>(inv + row_of[j] * H + h0);
      float *dst = alpha + (int64_t)h0 * ahs + e0 + j;
      dst[0] = v.x * w.x;
      dst[ahs] = v.y * w.y;
      dst[2 * ahs] = v.z * w.z;
      dst[3 * ahs] = v.w * w.w;
    }
  }
}

// Short rows (<= kTile entries): warp w owns rows w * RPW .. + RPW - 1 (RPW =
// 32 / H).  The rows' entries (contiguous in CSR) are staged in the warp's
// tile by cp.async, as many consecutive short rows at a time as fit (a
// BATCH), and the warp reduces them one row at a time: lane (part, h) takes
// entries part, part + P, ... of head h (P = 32 / H), an xor tree over the P
// parts finishes -- no lane waits on a longer row of another lane.  The row
// max of the fp64 scores is the score of the fp32 max of the stored values
// (LeakyReLU with slope >= 0 and IEEE rounding are monotone) -- exactly;
// slope < 0 takes the fp64 max of the scores.  kApply: the tile keeps
// exp(s - m), the batch's rows' 1 / S go to `inv`, and alpha = exp * (1 / S)
// is formed by the store.
template <int H, bool kScores, bool kApply>
__device__ __forceinline__ void stat_short_rows(float *T, uint8_t *row_of, float *inv, const int64_t *s_rp,
                                                int64_t rbase, int64_t n_rows, const int32_t *__restrict__ col,
                                                const float *__restrict__ el, const float *__restrict__ er,
                                                const float *logits, double slope, GatStat *__restrict__ st,
                                                float *alpha, int64_t ahs, int warp, int lane) {
  constexpr int kTile = kStatTileFloats / H;
  constexpr int RPW = 32 / H;
  constexpr int P = RPW;
  const int part = lane / H, h = lane % H;
  const int base = warp * RPW;  // CTA-local index of the warp's first row
  const double slope_l2e = slope * kLog2e;
  const int nr = (int)max((int64_t)0, min((int64_t)RPW, n_rows - (rbase + base)));
  // lane r (< nr) holds row r's start and end; batches are found by ballots
  const int64_t rp_lo = s_rp[base + min(lane, RPW)], rp_hi = s_rp[base + min(lane + 1, RPW)];
  const unsigned short_rows = __ballot_sync(0xffffffffu, lane < nr && rp_hi - rp_lo <= kTile);
  // el of the warp's rows, once: lane (r, h) holds el[row r][h]
  const float el_l = (kScores && part < nr) ? __ldg(el + (rbase + base + part) * H + h) : 0.0f;
  unsigned todo = short_rows;
  while (todo) {
    const int k = __ffs(todo) - 1;
    // rows k .. k2-1: consecutive short rows whose entries fit the tile
    const int64_t B0 = __shfl_sync(0xffffffffu, rp_lo, k);
    const unsigned fits = __ballot_sync(0xffffffffu, rp_hi - B0 <= kTile) & short_rows;
    const unsigned run = ~(fits >> k);  // first row >= k that does not fit / is not short
    const int k2 = k + (run ? __ffs(run) - 1 : 32 - k);
    todo &= ~(((k2 >= 32) ? 0xffffffffu : ((1u << k2) - 1u)));
    const int64_t B1 = __shfl_sync(0xffffffffu, rp_hi, k2 - 1);
    __syncwarp();
    stat_load<H, kScores>(T, B0, (int)(B1 - B0), col, er, logits, lane);
    __syncwarp();
    for (int q = k; q < k2; ++q) {
      const int64_t b = __shfl_sync(0xffffffffu, rp_lo, q);
      const int d = (int)(__shfl_sync(0xffffffffu, rp_hi, q) - b);
      if (d == 0) continue;
      float *Tr = T + (b - B0) * H + h;
      if (kApply && h == 0)
        for (int j = part; j < d; j += P) row_of[b - B0 + j] = (uint8_t)q;
      const double el_u = kScores ? (double)__shfl_sync(0xffffffffu, el_l, q * H + h) : 0.0;
      float mr = -INFINITY;
      {
        int j = part;
        for (; j + P < d; j += 2 * P) mr = fmaxf(mr, fmaxf(Tr[j * H], Tr[(j + P) * H]));
        if (j < d) mr = fmaxf(mr, Tr[j * H]);
      }
#pragma unroll
      for (int off = H; off < 32; off <<= 1) mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, off));
      double m = stat_score<kScores>(mr, el_u, slope);
      if (kScores && !(slope >= 0.0)) {
        m = -INFINITY;
        for (int j = part; j < d; j += P) m = fmax(m, stat_score<kScores>(Tr[j * H], el_u, slope));
#pragma unroll
        for (int off = H; off < 32; off <<= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
      }
      // exp(s - m) = 2^((s - m) log2 e): the argument is formed exactly enough
      // that its one rounding to fp32 dominates (<= |s - m| u), then ex2.approx
      // (<= 2 ulp).  Scores: s - m = x f - m with x = el + er exact in fp64 and
      // f = 1 or slope, so (s - m) log2e = fma(x, f log2e, -m log2e) in fp64.
      // Logits: t - t_max in fp32 is one rounding of the exact difference.
      // fp32 sums: every term is in (0, 1] and one is exactly 1 (the max), a
      // lane adds <= kTile / P = 32 of them -- relative error <= 37 u
      const double mm = m * kLog2e;
      auto ex_of = [&](float t) {
        float a;
        if (kScores) {
          const double x = el_u + (double)t;
          a = (float)fma(x, x >= 0.0 ? kLog2e : slope_l2e, -mm);
        } else {
          a = (t - mr) * (float)kLog2e;
        }
        return ex2_approx(a);
      };
      float sum = 0.0f;
      {
        int j = part;
        for (; j + P < d; j += 2 * P) {
          const float e0 = ex_of(Tr[j * H]), e1 = ex_of(Tr[(j + P) * H]);
          sum += e0;
          sum += e1;
          if (kApply) {
            Tr[j * H] = e0;  // own slots
            Tr[(j + P) * H] = e1;
          }
        }
        if (j < d) {
          const float e0 = ex_of(Tr[j * H]);
          sum += e0;
          if (kApply) Tr[j * H] = e0;
        }
      }
#pragma unroll
      for (int off = H; off < 32; off <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
      const float inv_s = __frcp_rn(sum);
      if (part == 0) {
        if (kApply) {
          inv[q * H + h] = inv_s;
        } else {
          GatStat g;
          g.m = m;
          g.inv_s = inv_s;
          g.pad = 0.f;
          st[(rbase + base + q) * H + h] = g;
        }
      }
    }
    if (kApply) {  // the batch's alpha (contiguous entries B0 .. B1) in 128-byte stores
      __syncwarp();
      stat_store_scaled<H>(T, row_of, inv, B0, (int)(B1 - B0), alpha, ahs, lane);
    }
  }
}

// Long rows (> kTile entries) are cut into tile-sized chunks; warp w takes
// chunks w, w + 8, ... and reduces them to a partial (m_w, s_w) with its OWN
// maximum m_w (s_w = sum of exp(s - m_w), fp64).  Warp k % 8 merges long row
// k's 8 partials in warp order -- M = max m_w, S = sum_w s_w exp(m_w - M)
// (fp64) -- after a named barrier the other warps only ARRIVE at, so they go
// on with the next long row and their short rows; only the alpha writes of a
// long row (kApply) wait (second named barrier) for its merged (M, S).
// Partials of up to kSlots long rows live in shared memory; a CTA with more
// long rows processes them in batches separated by a CTA barrier.
// Slots: <= 8 KB of partials (48 KB static smem) and one named barrier per
// long row (two with kApply) out of the 15 a CTA has besides barrier 0.
template <int H, bool kApply>
struct StatSlots {
  static constexpr int kMem = (64 / H) < 16 ? (64 / H) : 16;
  static constexpr int kBar = kApply ? 7 : 15;
  static constexpr int kSlots = kMem < kBar ? kMem : kBar;
};

// named CTA barriers (bar.sync / bar.arrive over `n` threads): the warps that
// produce a long row's partials arrive without waiting; only the warp that
// merges them (and, with kApply, the warps that then need the merged result)
// wait -- ordered for the memory model and for compute-sanitizer's racecheck
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

#if GSP_STAT_TRACE
// tuning probe only (-DGSP_STAT_TRACE): per CTA start / end (globaltimer, ns),
// SM id and long-row count of the last row_stats_warp launch
constexpr int kTraceMax = 1 << 16;
__device__ unsigned long long g_stat_trace[4][kTraceMax];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif
template <int H, bool kScores, bool kApply>
__global__ void __launch_bounds__(kStatWarps * 32, GSP_STAT_MINB) row_stats_warp(const int64_t *__restrict__ rp,
                                                                  const int32_t *__restrict__ col,
                                                                  const float *__restrict__ el,
                                                                  const float *__restrict__ er, const float *logits,
                                                                  double slope, int64_t n_rows,
                                                                  GatStat *__restrict__ st, float *alpha,
                                                                  int64_t ahs) {
  constexpr int kTile = kStatTileFloats / H;
  constexpr int kRows = kStatWarps * (32 / H);  // rows per CTA (32 / H per warp: lane = (row, head))
  constexpr int kSlots = StatSlots<H, kApply>::kSlots;
  constexpr int P = 32 / H;
  __shared__ __align__(16) float s_tile[kStatWarps][kStatTileFloats];
  __shared__ double s_pm[kSlots][kStatWarps][H];  // partial max (score) per slot, warp, head
  __shared__ double s_ps[kSlots][kStatWarps][H];  // partial sum of exp(s - m_w)
  __shared__ double s_M[kSlots][H];               // merged max (kApply)
  __shared__ float s_inv[kSlots][H];              // merged 1 / S (kApply)
  __shared__ int64_t s_rp[kRows + 1];
  __shared__ uint8_t s_rowof[kApply ? kStatWarps : 1][kApply ? kTile : 1];            // batch row of an entry
  __shared__ __align__(16) float s_invw[kApply ? kStatWarps : 1][kApply ? 32 : 1];   // 1 / S per (batch row, head)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int h = lane % H, part = lane / H;
  const double slope_l2e = slope * kLog2e;
  const int64_t rbase = (int64_t)blockIdx.x * kRows;
#if GSP_STAT_TRACE
  if (tid == 0 && blockIdx.x < kTraceMax) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_stat_trace[0][blockIdx.x] = gtimer();
    g_stat_trace[2][blockIdx.x] = smid;
  }
  struct TraceEnd {
    int lane;
    __device__ ~TraceEnd() {
      if (lane == 0 && blockIdx.x < kTraceMax) atomicMax(&g_stat_trace[1][blockIdx.x], gtimer());
    }
  } trace_end{(int)(threadIdx.x & 31)};
#endif
  // the CTA's row pointers and its long rows, once (nobody is busy yet)
  for (int i = tid; i <= kRows; i += kStatWarps * 32) s_rp[i] = __ldg(rp + min(rbase + i, n_rows));
  __syncthreads();
  // every warp finds the CTA's long rows itself (ballots over s_rp): no second
  // CTA barrier before the warps start working
  constexpr int kMasks = (kRows + 31) / 32;
  unsigned lm[kMasks];
  int nlong = 0;
#pragma unroll
  for (int q = 0; q < kMasks; ++q) {
    const int r = q * 32 + lane;
    lm[q] = __ballot_sync(0xffffffffu, r < kRows && (s_rp[r + 1] - s_rp[r]) > kTile);
    nlong += __popc(lm[q]);
  }
#if GSP_STAT_TRACE
  if (tid == 0 && blockIdx.x < kTraceMax) g_stat_trace[3][blockIdx.x] = nlong;
#endif
  auto long_row = [&](int k) {  // CTA-local index of the k-th long row (index order)
#pragma unroll
    for (int q = 0; q < kMasks; ++q) {
      const int c = __popc(lm[q]);
      if (k < c) return q * 32 + (int)__fns(lm[q], 0, k + 1);
      k -= c;
    }
    return 0;
  };
  float *T = s_tile[warp];
  // ---- 1. long rows: per-warp partials, merged by the last warp to arrive
  for (int k0 = 0; k0 < nlong; k0 += kSlots) {
    const int kn = min(kSlots, nlong - k0);
    if (k0 > 0) __syncthreads();  // slots and barrier ids are reused: the previous batch is complete
    for (int k = 0; k < kn; ++k) {
      const int lr = long_row(k0 + k);
      const int64_t r = rbase + lr, b = s_rp[lr], e1 = s_rp[lr + 1];
      const double el_u = kScores ? (double)__ldg(el + r * H + h) : 0.0;
      double m = -INFINITY, sum = 0.0;
      for (int64_t c0 = b + (int64_t)warp * kTile; c0 < e1; c0 += (int64_t)kStatWarps * kTile) {
        const int cnt = (int)min((int64_t)kTile, e1 - c0);
        __syncwarp();
        stat_load<H, kScores>(T, c0, cnt, col, er, logits, lane);
        __syncwarp();
        float mr = -INFINITY;  // exact chunk max of the scores via the stored values (monotone, see stat_row)
        for (int j = part; j < cnt; j += P) mr = fmaxf(mr, T[j * H + h]);
#pragma unroll
        for (int off = H; off < 32; off <<= 1) mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, off));
        double mc = stat_score<kScores>(mr, el_u, slope);
        if (kScores && !(slope >= 0.0)) {
          mc = -INFINITY;
          for (int j = part; j < cnt; j += P) mc = fmax(mc, stat_score<kScores>(T[j * H + h], el_u, slope));
#pragma unroll
          for (int off = H; off < 32; off <<= 1) mc = fmax(mc, __shfl_xor_sync(0xffffffffu, mc, off));
        }
        float scf = 0.0f;  // <= kTile / P = 32 terms in (0, 1] per lane (as the short rows)
        for (int j = part; j < cnt; j += P) scf += stat_exp<kScores>(T[j * H + h], el_u, slope_l2e, mc);
#pragma unroll
        for (int off = H; off < 32; off <<= 1) scf += __shfl_xor_sync(0xffffffffu, scf, off);
        const double sc = (double)scf;
        // fold the chunk into the warp's partial (chunks in increasing order)
        if (mc > m) {
          sum = (m == -INFINITY) ? sc : sum * exp(m - mc) + sc;
          m = mc;
        } else if (mc != -INFINITY) {
          sum += sc * exp(mc - m);
        } else {
          sum += sc;  // NaN propagates; empty chunks do not occur
        }
      }
      if (part == 0) {
        s_pm[k][warp][h] = m;
        s_ps[k][warp][h] = sum;
      }
      __syncwarp();
      const int bar_merge = 1 + (kApply ? 2 * k : k);
      if (warp != k % kStatWarps) {
        named_arrive(bar_merge, kStatWarps * 32);
        continue;
      }
      named_sync(bar_merge, kStatWarps * 32);  // every warp's partial of row k is written
      if (lane < H) {  // merge the 8 partials in warp order
        double M = -INFINITY;
        for (int w = 0; w < kStatWarps; ++w) M = fmax(M, s_pm[k][w][lane]);
        double S = 0.0;
        for (int w = 0; w < kStatWarps; ++w) {
          const double mw = s_pm[k][w][lane];
          if (mw != -INFINITY) S += s_ps[k][w][lane] * exp(mw - M);
          else S += s_ps[k][w][lane];
        }
        if (kApply) {
          s_M[k][lane] = M;
          s_inv[k][lane] = (float)(1.0 / S);
        } else {
          GatStat g;
          g.m = M;
          g.inv_s = (float)(1.0 / S);
          g.pad = 0.f;
          st[r * H + lane] = g;
        }
      }
      if (kApply) {
        __syncwarp();
        named_arrive(bar_merge + 1, kStatWarps * 32);  // (M, 1/S) of row k published
      }
    }
    // ---- 2. short rows (first batch only), while the other warps finish their long chunks
    if (k0 == 0) stat_short_rows<H, kScores, kApply>(T, s_rowof[kApply ? warp : 0], s_invw[kApply ? warp : 0], s_rp, rbase, n_rows, col, el, er, logits, slope, st, alpha, ahs, warp, lane);
    // ---- 3. kApply: alpha of this batch's long rows, once their (M, S) are merged
    if (kApply) {
      for (int k = 0; k < kn; ++k) {
        const int lr = long_row(k0 + k);
        const int64_t r = rbase + lr, b = s_rp[lr], e1 = s_rp[lr + 1];
        // every warp but the merging one meets the publishing warp here (even
        // without a chunk of the row: the barrier counts all 8 warps)
        if (warp != k % kStatWarps) named_sync(1 + 2 * k + 1, kStatWarps * 32);
        if (b + (int64_t)warp * kTile >= e1) continue;
        const double el_u = kScores ? (double)__ldg(el + r * H + h) : 0.0;
        const double M = s_M[k][h];
        const float inv_s = s_inv[k][h];
        for (int64_t c0 = b + (int64_t)warp * kTile; c0 < e1; c0 += (int64_t)kStatWarps * kTile) {
          const int cnt = (int)min((int64_t)kTile, e1 - c0);
          __syncwarp();
          stat_load<H, kScores>(T, c0, cnt, col, er, logits, lane);
          __syncwarp();
          for (int j = part; j < cnt; j += P)
            T[j * H + h] = stat_exp<kScores>(T[j * H + h], el_u, slope_l2e, M) * inv_s;
          __syncwarp();
          stat_store_alpha<H>(T, c0, cnt, alpha, ahs, lane);
        }
      }
    }
  }
  if (nlong == 0) stat_short_rows<H, kScores, kApply>(T, s_rowof[kApply ? warp : 0], s_invw[kApply ? warp : 0], s_rp, rbase, n_rows, col, el, er, logits, slope, st, alpha, ahs, warp, lane);
}

// Fallback for H not dividing 32: one thread per (row, head), sequential.
template <bool kScores, bool kApply>
__global__ void row_stats_thread(const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                                 const float *__restrict__ el, const float *__restrict__ er, const float *logits,
                                 double slope, int H, int64_t n_rows, GatStat *__restrict__ st, float *alpha,
                                 int64_t ahs) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_rows * H) return;
  const int64_t r = t / H;
  const int h = (int)(t % H);
  const int64_t b = rp[r], e1 = rp[r + 1];
  if (b == e1) return;
  const double el_u = kScores ? (double)el[r * H + h] : 0.0;
  auto score = [&](int64_t e) -> double {
    if (kScores) {
      const double x = el_u + (double)er[(int64_t)col[e] * H + h];
      return x >= 0.0 ? x : slope * x;
    } else {
      return (double)logits[e * H + h];
    }
  };
  double m = -INFINITY;
  for (int64_t e = b; e < e1; ++e) m = fmax(m, score(e));
  double s = 0.0;
  for (int64_t e = b; e < e1; ++e) s += (double)expf((float)(score(e) - m));
  if (kApply) {
    const float inv_s = (float)(1.0 / s);
    for (int64_t e = b; e < e1; ++e) alpha[ahs ? h * ahs + e : e * H + h] = expf((float)(score(e) - m)) * inv_s;
    return;
  }
  GatStat g;
  g.m = m;
  g.inv_s = (float)(1.0 / s);
  g.pad = 0.f;
  st[t] = g;
}

template <bool kScores, bool kApply>
static gsp_status launch_stats(const gsp_csr *a, const float *el, const float *er, const float *logits, double slope,
                               int H, GatStat *st, float *alpha, cudaStream_t s, int64_t ahs = 0) {
  if (a->n_rows == 0) return GSP_OK;
  const float *vsrc = kScores ? er : logits;
  const bool vec_ok = H < 4 ? (H == 1 || aligned8(vsrc)) : aligned16(vsrc);
  if (32 % H == 0 && (vec_ok || !kScores)) {
    const unsigned blocks = (unsigned)ceil_div(a->n_rows, kStatWarps * (32 / H));
#define GSP_STATS_H(HH)                                                                                       \
  case HH:                                                                                                   \
    row_stats_warp<HH, kScores, kApply><<<blocks, kStatWarps * 32, 0, s>>>(a->row_ptr, a->col_idx, el, er,     \
                                                                         logits, slope, a->n_rows, st, alpha, ahs); \
    break;
    switch (H) {
      GSP_STATS_H(1) GSP_STATS_H(2) GSP_STATS_H(4) GSP_STATS_H(8) GSP_STATS_H(16) GSP_STATS_H(32)
    }
#undef GSP_STATS_H
  } else {
    const int64_t blocks = ceil_div(a->n_rows * H, 256);
    row_stats_thread<kScores, kApply><<<(unsigned)blocks, 256, 0, s>>>(a->row_ptr, a->col_idx, el, er, logits,
                                                                        slope, H, a->n_rows, st, alpha, ahs);
  }
  return check_launch("row_stats");
}

// alpha = softmax_row(LeakyReLU(el[u] + er[v])) written per entry and head
// (the GAT backward recomputes alpha with the same reductions as the forward)
gsp_status launch_row_softmax_scores(const gsp_csr *a, const float *el, const float *er, double slope, int H,
                                     float *alpha, cudaStream_t s) {
  return launch_stats<true, true>(a, el, er, nullptr, slope, H, nullptr, alpha, s);
}

// ------------------------------------------------------------------------
// Attention projection el/er (a4).  One warp per row.  When a head's D/V
// vectors tile the warp (32 % (D/V) == 0) lanes cover several heads at once
// and reduce with a segmented xor tree; otherwise heads are looped.
// ------------------------------------------------------------------------
template <int V>
__global__ void __launch_bounds__(256) attn_project_warp(int64_t n, int H, int64_t D, const float *__restrict__ z,
                                                         int64_t ldz, const float *__restrict__ al,
                                                         const float *__restrict__ ar, float *__restrict__ el,
                                                         float *__restrict__ er) {
  const int64_t u = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (u >= n) return;
  const int lane = threadIdx.x & 31;
  const int64_t VH = D / V;  // vectors per head
  const float *zu = z + u * ldz;
  if (VH <= 32 && 32 % VH == 0) {
    const int64_t nvec = (int64_t)H * VH;
    for (int64_t base = 0; base < nvec; base += 32) {
      const int64_t k = base + lane;
      float sl = 0.f, sr = 0.f;
      if (k < nvec) {
        float zv[V], lv[V], rv[V];
        Vec<V>::ld(zv, zu + k * V);
        Vec<V>::ld(lv, al + k * V);
        Vec<V>::ld(rv, ar + k * V);
#pragma unroll
        for (int i = 0; i < V; ++i) {
          sl = fmaf(lv[i], zv[i], sl);
          sr = fmaf(rv[i], zv[i], sr);
        }
      }
      for (int off = 1; off < VH; off <<= 1) {
        sl += __shfl_xor_sync(0xffffffffu, sl, off);
        sr += __shfl_xor_sync(0xffffffffu, sr, off);
      }
      if (k < nvec && (lane % VH) == 0) {
        const int64_t h = k / VH;
        el[u * H + h] = sl;
        er[u * H + h] = sr;
      }
    }
  } else {
    for (int h = 0; h < H; ++h) {
      float sl = 0.f, sr = 0.f;
      for (int64_t k = lane; k < VH; k += 32) {
        float zv[V], lv[V], rv[V];
        Vec<V>::ld(zv, zu + (h * VH + k) * V);
        Vec<V>::ld(lv, al + (h * VH + k) * V);
        Vec<V>::ld(rv, ar + (h * VH + k) * V);
#pragma unroll
        for (int i = 0; i < V; ++i) {
          sl = fmaf(lv[i], zv[i], sl);
          sr = fmaf(rv[i], zv[i], sr);
        }
      }
      for (int off = 16; off > 0; off >>= 1) {
        sl += __shfl_xor_sync(0xffffffffu, sl, off);
        sr += __shfl_xor_sync(0xffffffffu, sr, off);
      }
      if (lane == 0) {
        el[u * H + h] = sl;
        er[u * H + h] = sr;
      }
    }
  }
}

// Streaming form for the common layout (float4 vectors, a head = VH vectors
// with VH | 32, H*D <= 32*4*NV): each warp owns kAPR consecutive rows, issues
// every Z load of its rows before the first use (NV float4 per lane per row),
// keeps a_l / a_r in registers, then reduces each head with a segmented xor
// tree.  Same per-(row, head) order as attn_project_warp (lane-sequential fma
// over V, then the xor tree).
constexpr int kAPR = 2;  // rows per warp
template <int NV>
__global__ void __launch_bounds__(256) attn_project_stream(int64_t n, int H, int VH, const float *__restrict__ z,
                                                           int64_t ldz, const float *__restrict__ al,
                                                           const float *__restrict__ ar, float *__restrict__ el,
                                                           float *__restrict__ er) {
  const int lane = threadIdx.x & 31;
  const int64_t u0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * kAPR;
  if (u0 >= n) return;
  const int nvec = H * VH;
  float4 a[NV], b[NV], zv[kAPR][NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int k = lane + 32 * i;
    a[i] = k < nvec ? __ldg(reinterpret_cast<const float4 *>(al) + k) : make_float4(0, 0, 0, 0);
    b[i] = k < nvec ? __ldg(reinterpret_cast<const float4 *>(ar) + k) : make_float4(0, 0, 0, 0);
  }
#pragma unroll
  for (int r = 0; r < kAPR; ++r) {
    const int64_t u = u0 + r;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int k = lane + 32 * i;
      zv[r][i] = (u < n && k < nvec) ? __ldg(reinterpret_cast<const float4 *>(z + u * ldz) + k) : make_float4(0, 0, 0, 0);
    }
  }
#pragma unroll
  for (int r = 0; r < kAPR; ++r) {
    const int64_t u = u0 + r;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const float4 q = zv[r][i];
      float sl = fmaf(a[i].w, q.w, fmaf(a[i].z, q.z, fmaf(a[i].y, q.y, a[i].x * q.x)));
      float sr = fmaf(b[i].w, q.w, fmaf(b[i].z, q.z, fmaf(b[i].y, q.y, b[i].x * q.x)));
      for (int off = 1; off < VH; off <<= 1) {
        sl += __shfl_xor_sync(0xffffffffu, sl, off);
        sr += __shfl_xor_sync(0xffffffffu, sr, off);
      }
      const int k = lane + 32 * i;
      if (u < n && k < nvec && (lane % VH) == 0) {
        const int64_t h = k / VH;
        el[u * H + h] = sl;
        er[u * H + h] = sr;
      }
    }
  }
}

}  // namespace gsp

using namespace gsp;

extern "C" gsp_status gsp_edge_softmax(const gsp_csr *a, int32_t heads, const float *logits, float *alpha,
                                       gsp_stream stream) {
  const char *fn = "gsp_edge_softmax";
  clear_detail();
  gsp_status st = check_csr(a, false, fn);
  if (st) return st;
  if (heads <= 0) return fail(GSP_ERR_INVALID_ARG, "%s: heads must be >= 1", fn);
  if (a->nnz == 0 || a->n_rows == 0) return GSP_OK;
  if (!logits || !alpha) return fail(GSP_ERR_INVALID_ARG, "%s: null pointer", fn);
  const size_t bytes = (size_t)a->nnz * heads * 4;
  if (logits != alpha && overlaps(logits, bytes, alpha, bytes))
    return fail(GSP_ERR_ALIAS, "%s: logits and alpha partially overlap", fn);
  if (validate_mode()) {
    const float *arr[1] = {logits};
    const int64_t cnt[1] = {a->nnz * heads};
    const char *nm[1] = {"logits"};
    if ((st = check_finite(cs(stream), fn, 1, arr, cnt, nm))) return st;
  }
  return launch_stats<false, true>(a, nullptr, nullptr, logits, 0.0, heads, nullptr, alpha, cs(stream));
}

extern "C" gsp_status gsp_attn_project(int64_t n, int32_t heads, int64_t d, const float *z, int64_t ldz,
                                       const float *a_l, const float *a_r, float *el, float *er, gsp_stream stream) {
  const char *fn = "gsp_attn_project";
  clear_detail();
  if (n < 0 || heads <= 0 || d < 0 || ldz < (int64_t)heads * d)
    return fail(GSP_ERR_INVALID_ARG, "%s: bad sizes", fn);
  if (n == 0) return GSP_OK;
  if (!z || !a_l || !a_r || !el || !er) return fail(GSP_ERR_INVALID_ARG, "%s: null pointer", fn);
  if (n >= (int64_t(1) << 31)) return fail(GSP_ERR_UNSUPPORTED, "%s: n must be < 2^31", fn);
  const unsigned blocks = (unsigned)ceil_div(n, 8);
  cudaStream_t s = cs(stream);
  const int64_t VH = d / 4, nvec = (int64_t)heads * VH;
  const bool vec = d % 4 == 0 && ldz % 4 == 0 && aligned16(z) && aligned16(a_l) && aligned16(a_r);
  if (vec && VH >= 1 && VH <= 32 && 32 % VH == 0 && nvec <= 32 * 4) {
    const unsigned sb = (unsigned)ceil_div(n, 8 * kAPR);
    if (nvec <= 32) attn_project_stream<1><<<sb, 256, 0, s>>>(n, heads, (int)VH, z, ldz, a_l, a_r, el, er);
    else if (nvec <= 64) attn_project_stream<2><<<sb, 256, 0, s>>>(n, heads, (int)VH, z, ldz, a_l, a_r, el, er);
    else attn_project_stream<4><<<sb, 256, 0, s>>>(n, heads, (int)VH, z, ldz, a_l, a_r, el, er);
  } else if (vec)
    attn_project_warp<4><<<blocks, 256, 0, s>>>(n, heads, d, z, ldz, a_l, a_r, el, er);
  else
    attn_project_warp<1><<<blocks, 256, 0, s>>>(n, heads, d, z, ldz, a_l, a_r, el, er);
  return check_launch("attn_project");
}

// alpha head-major [H][ahs] for the two-launch staged schedule: ahs = nnz rounded
// up to 32 entries, so every head's run starts 128-byte aligned (TMA bulk copies)
static int64_t gat_ahs(const gsp_csr *a) { return (std::max<int64_t>(a->nnz, 1) + 31) / 32 * 32; }
static size_t gat_hm_bytes(const gsp_csr *a, int heads) { return (size_t)gat_ahs(a) * heads * 4; }
static size_t gat_stat_bytes(const gsp_csr *a, int heads) {
  return (size_t)std::max<int64_t>(a->n_rows, 0) * heads * sizeof(GatStat);  // (m, 1/S) per (row, head)
}

extern "C" gsp_status gsp_gat_workspace(const gsp_csr *a, int32_t heads, size_t *ws_bytes) {
  clear_detail();
  if (!a || heads <= 0 || !ws_bytes) return fail(GSP_ERR_INVALID_ARG, "gsp_gat_workspace: bad argument");
  *ws_bytes = std::max(gat_stat_bytes(a, heads), gat_hm_bytes(a, heads));
  return GSP_OK;
}

static gsp_status gat_aggregate_impl(const gsp_csr *a, int32_t heads, const float *el, const float *er,
                                     double negative_slope, const float *z, int64_t d, int64_t ldz, float *y,
                                     int64_t ldy, float *alpha_out, const float *bias, int act, void *ws,
                                     size_t ws_bytes, cudaStream_t s, const char *fn) {
  clear_detail();
  gsp_status st = check_csr(a, false, fn);
  if (st) return st;
  if (heads <= 0 || d < 0) return fail(GSP_ERR_INVALID_ARG, "%s: heads >= 1 and d >= 0 required", fn);
  const int64_t f = (int64_t)heads * d;
  if (ldz < f || ldy < f) return fail(GSP_ERR_INVALID_ARG, "%s: need ldz, ldy >= heads*d", fn);
  if (a->n_rows == 0 || f == 0) return GSP_OK;
  if (!y || !el || (a->n_cols > 0 && (!z || !er)))
    return fail(GSP_ERR_INVALID_ARG, "%s: null pointer", fn);
  const size_t zb = a->n_cols ? (size_t)((a->n_cols - 1) * ldz + f) * 4 : 0;
  const size_t yb = (size_t)((a->n_rows - 1) * ldy + f) * 4;
  if (overlaps(z, zb, y, yb)) return fail(GSP_ERR_ALIAS, "%s: z and y overlap", fn);
  if (validate_mode()) {  // the score inputs el / er must be finite
    const float *arr[2] = {el, er};
    const int64_t cnt[2] = {a->n_rows * heads, a->n_cols * heads};
    const char *nm[2] = {"el", "er"};
    if ((st = check_finite(s, fn, 2, arr, cnt, nm))) return st;
  }
  int vmax = 1;
  if (ldz % 4 == 0 && aligned16(z)) vmax = 4;
  else if (ldz % 2 == 0 && aligned8(z)) vmax = 2;
  // two launches when the workspace can hold the statistics (row_stats_warp
  // for all heads, then the aggregate, several whole heads per team);
  // otherwise one launch with the statistics reduced inside the aggregate
  // kernel, one head per team (fp64 row state in registers)
  //   three schedules, by workspace:
  //  * >= gat_hm_bytes (the size gsp_gat_workspace reports), no alpha_out:
  //    the statistics launch writes alpha head-major [H][ahs]; the aggregate
  //    stages the slab's heads of it with the CSR window (TMA) and gathers
  //    with weights read from shared memory (WeightAlphaHM);
  //  * >= gat_stat_bytes: statistics (m, 1/S) only, alpha formed in the
  //    aggregate (WeightGatPre) -- also the schedule that writes alpha_out;
  //  * otherwise one launch (WeightGat).
  const bool hm = ws && ws_bytes >= gat_hm_bytes(a, heads) && reinterpret_cast<uintptr_t>(ws) % 128 == 0 &&
                  !alpha_out && 32 % heads == 0 && aligned16(a->col_idx) && a->nnz > 0;
  const bool pre = !hm && ws && ws_bytes >= gat_stat_bytes(a, heads) && aligned16(ws) && 32 % heads == 0;
  EngineLaunch L;
  st = engine_plan(a->n_rows, a->n_cols, a->nnz, f, d, vmax, 0, 0, &L, (pre || hm) ? kMaxHpt : 1);
  if (st) return st;
  if (hm) {
    // keep the staged window (col + hpt weight runs) within ~42 KB so four
    // CTAs still fit on an SM (the 64-register budget allows four)
    const int hpt = engine_hpt(L, d, heads);
    const int64_t win_max = 43008 / (4 * (1 + hpt));
    int64_t c = ((win_max - kHub - 8) / 512) * 512;
    if (c < 512) c = 512;
    if (c < L.block_nnz) {
      st = engine_plan(a->n_rows, a->n_cols, a->nnz, f, d, vmax, 0, (int32_t)c, &L, kMaxHpt);
      if (st) return st;
    }
  }
  EngineParams p;
  p.row_ptr = a->row_ptr;
  p.col = a->col_idx;
  p.x = z;
  p.y = y;
  p.n_rows = a->n_rows;
  p.ldx = ldz;
  p.ldy = ldy;
  p.f = f;
  p.block_nnz = L.block_nnz;
  p.nblk = L.nblk;
  p.head_dim = d;
  p.y_vec_ok = engine_y_vec_ok(L, y, ldy);
  engine_stage(p, L, a->nnz, a->col_idx, nullptr);
  p.hpt = engine_hpt(L, d, heads);
  p.bias = bias;
  p.act = act;
  if ((st = engine_ldxv(p, L, a->n_cols, ldz))) return st;
  if (hm) {
    float *alpha_hm = static_cast<float *>(ws);
    const int64_t ahs = gat_ahs(a);
    if ((st = launch_stats<true, true>(a, el, er, nullptr, negative_slope, heads, nullptr, alpha_hm, s, ahs)))
      return st;
    if (p.stage) {
      p.stage_hm = alpha_hm;
      p.stage_hm_stride = ahs;
      p.stage_heads = p.hpt;
    }
    return engine_launch(L, p, WeightAlphaHM{alpha_hm, ahs}, s);
  }
  if (pre) {
    GatStat *stat = static_cast<GatStat *>(ws);
    if ((st = launch_stats<true, false>(a, el, er, nullptr, negative_slope, heads, stat, nullptr, s))) return st;
    WeightGatPre w{el, er, alpha_out, negative_slope, heads, stat};
    return engine_launch(L, p, w, s);
  }
  WeightGat w{el, er, alpha_out, negative_slope, heads, nullptr};
  return engine_launch(L, p, w, s);
}

extern "C" gsp_status gsp_gat_aggregate(const gsp_csr *a, int32_t heads, const float *el, const float *er,
                                        double negative_slope, const float *z, int64_t d, int64_t ldz, float *y,
                                        int64_t ldy, float *alpha_out, void *ws, size_t ws_bytes, gsp_stream stream) {
  return gat_aggregate_impl(a, heads, el, er, negative_slope, z, d, ldz, y, ldy, alpha_out, nullptr, 0, ws, ws_bytes,
                            cs(stream), "gsp_gat_aggregate");
}

extern "C" gsp_status gsp_gat_aggregate_bias_act(const gsp_csr *a, int32_t heads, const float *el, const float *er,
                                                 double negative_slope, const float *z, int64_t d, int64_t ldz,
                                                 const float *bias, gsp_act act, float *y, int64_t ldy, void *ws,
                                                 size_t ws_bytes, gsp_stream stream) {
  if (act < GSP_ACT_NONE || act > GSP_ACT_ELU) return fail(GSP_ERR_INVALID_ARG, "gsp_gat_aggregate_bias_act: bad act");
  return gat_aggregate_impl(a, heads, el, er, negative_slope, z, d, ldz, y, ldy, nullptr, bias, (int)act, ws, ws_bytes,
                            cs(stream), "gsp_gat_aggregate_bias_act");
}

#if GSP_STAT_TRACE
extern "C" int gsp_debug_stat_trace(void *dst, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(dst, gsp::g_stat_trace, std::min(bytes, sizeof(gsp::g_stat_trace)));
}
extern "C" int gsp_debug_stat_trace_reset() {
  static unsigned long long zero[4][gsp::kTraceMax];
  return (int)cudaMemcpyToSymbol(gsp::g_stat_trace, zero, sizeof(zero));
}
#endif
