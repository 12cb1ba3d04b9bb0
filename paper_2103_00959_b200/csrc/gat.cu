// gat.cu -- GAT path: attention projection (a4), edge softmax (a6) and the
// fused score -> softmax -> multi-head SpMM aggregate (a5+a6+a7).
// PAPER.md P:253 (GAT), P:648-649 (multi-head SpMM), P:653-656 (edge-wise
// softmax with warp-level max / sum reductions); readings A9-A14.
#include "spmm_engine.cuh"

#ifndef GSP_HM_WIN_BYTES
#define GSP_HM_WIN_BYTES 43008
#endif

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
#ifndef GSP_STAT_LONG_SLICE
#define GSP_STAT_LONG_SLICE 128
#endif
constexpr int kLongSlice = GSP_STAT_LONG_SLICE;  // rows a long CTA scans for long rows (<= 256)
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
      if (kApply)
        for (int j = lane; j < d; j += 32) row_of[b - B0 + j] = (uint8_t)q;
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
// Long rows (> kTile entries) of a long CTA's slice, kSlots at a time: the
// group's chunks (kTile entries each) are numbered back to back, c = pre_k + j
// for chunk j of row k, and warp w takes c = w, w + 8, ...  Chunk j belongs to
// RESIDUE q = j % 8 of its row; whichever warp computes it (w = (pre_k + j) % 8)
// folds the row's residue-q chunks in increasing j into a partial with its own
// max m_q (s_q = sum of exp(s - m_q), fp64), and the residues are merged in q
// order -- M = max m_q, S = sum_q s_q exp(m_q - M) -- so the order depends on
// the row alone.  kApply then writes alpha chunk by chunk the same way.
template <int H>
struct LongSlots {
  static constexpr int kSlots = (32 / H) > 8 ? 8 : ((32 / H) > 1 ? 32 / H : 1);  // rows per group (<= 2 KB of partials per array)
};

template <int H, bool kScores, bool kApply>
__device__ __forceinline__ void stat_long_group(float *T, double (*s_pm)[kStatWarps][H],
                                                double (*s_ps)[kStatWarps][H], double (*s_M)[H], float (*s_inv)[H],
                                                const int64_t *s_lr, const int64_t *s_lb, const int *s_pre, int nk,
                                                const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                                                const float *__restrict__ el, const float *__restrict__ er,
                                                const float *logits, double slope, double slope_l2e,
                                                GatStat *__restrict__ st, float *alpha, int64_t ahs, int warp,
                                                int lane, int tid) {
  constexpr int kTile = kStatTileFloats / H;
  constexpr int P = 32 / H;
  const int h = lane % H, part = lane / H;
  for (int i = tid; i < nk * kStatWarps * H; i += kStatWarps * 32) {
    (&s_pm[0][0][0])[i] = -INFINITY;
    (&s_ps[0][0][0])[i] = 0.0;
  }
  __syncthreads();
  const int total = s_pre[nk];
  int k = 0;
  double m = -INFINITY, sum = 0.0;  // running partial of (row k, this warp's residue)
  auto flush = [&]() {
    if (m != -INFINITY || sum != 0.0) {
      const int q = (int)(((warp - s_pre[k]) % kStatWarps + kStatWarps) % kStatWarps);
      if (part == 0) {
        s_pm[k][q][h] = m;
        s_ps[k][q][h] = sum;
      }
    }
    m = -INFINITY;
    sum = 0.0;
  };
  double el_u = 0.0;
  int el_k = -1;
  for (int c = warp; c < total; c += kStatWarps) {
    int kk = k;
    while (kk + 1 < nk && s_pre[kk + 1] <= c) ++kk;
    if (kk != k) {
      flush();
      k = kk;
    }
    if (kScores && el_k != k) {
      el_u = (double)__ldg(el + s_lr[k] * H + h);
      el_k = k;
    }
    const int64_t e1 = s_lb[k + 1 + nk];  // row end (see caller's layout)
    const int64_t c0 = s_lb[k] + (int64_t)(c - s_pre[k]) * kTile;
    const int cnt = (int)min((int64_t)kTile, e1 - c0);
    __syncwarp();
    stat_load<H, kScores>(T, c0, cnt, col, er, logits, lane);
    __syncwarp();
    float mr = -INFINITY;  // exact chunk max of the scores via the stored values (monotone)
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
    // fold the chunk into the residue's partial (its chunks in increasing order)
    if (mc > m) {
      sum = (m == -INFINITY) ? sc : sum * exp(m - mc) + sc;
      m = mc;
    } else if (mc != -INFINITY) {
      sum += sc * exp(mc - m);
    } else {
      sum += sc;  // NaN propagates; empty chunks do not occur
    }
  }
  if (total > warp) flush();
  __syncthreads();
  for (int i = tid; i < nk * H; i += kStatWarps * 32) {  // merge the residues in order
    const int kq = i / H, hh = i % H;
    double M = -INFINITY;
    for (int q = 0; q < kStatWarps; ++q) M = fmax(M, s_pm[kq][q][hh]);
    double S = 0.0;
    for (int q = 0; q < kStatWarps; ++q) {
      const double mq = s_pm[kq][q][hh];
      if (mq != -INFINITY) S += s_ps[kq][q][hh] * exp(mq - M);
      else S += s_ps[kq][q][hh];
    }
    if (kApply) {
      s_M[kq][hh] = M;
      s_inv[kq][hh] = (float)(1.0 / S);
    } else {
      GatStat g;
      g.m = M;
      g.inv_s = (float)(1.0 / S);
      g.pad = 0.f;
      st[s_lr[kq] * H + hh] = g;
    }
  }
  __syncthreads();
  if (kApply) {
    k = 0;
    el_k = -1;
    for (int c = warp; c < total; c += kStatWarps) {
      while (k + 1 < nk && s_pre[k + 1] <= c) ++k;
      if (kScores && el_k != k) {
        el_u = (double)__ldg(el + s_lr[k] * H + h);
        el_k = k;
      }
      const int64_t e1 = s_lb[k + 1 + nk];
      const int64_t c0 = s_lb[k] + (int64_t)(c - s_pre[k]) * kTile;
      const int cnt = (int)min((int64_t)kTile, e1 - c0);
      const double M = s_M[k][h];
      const float inv_s = s_inv[k][h];
      __syncwarp();
      stat_load<H, kScores>(T, c0, cnt, col, er, logits, lane);
      __syncwarp();
      for (int j = part; j < cnt; j += P) T[j * H + h] = stat_exp<kScores>(T[j * H + h], el_u, slope_l2e, M) * inv_s;
      __syncwarp();
      stat_store_alpha<H>(T, c0, cnt, alpha, ahs, lane);
    }
  }
  __syncthreads();  // the group's shared arrays are rewritten by the next group
}

// Grid: n_long LONG CTAs first, then the SHORT CTAs.
//  * long CTA c scans rows [c * long_rows, (c + 1) * long_rows) for rows of
//    more than kTile entries and reduces each with the whole CTA (they start
//    first, so the power-law tail overlaps the bulk of the short rows);
//  * short CTA b owns rows [b * kRows, (b + 1) * kRows) and reduces their
//    short rows, warp by warp (stat_short_rows); its long rows are skipped.
template <int H, bool kScores, bool kApply>
__global__ void __launch_bounds__(kStatWarps * 32, GSP_STAT_MINB) row_stats_warp(const int64_t *__restrict__ rp,
                                                                  const int32_t *__restrict__ col,
                                                                  const float *__restrict__ el,
                                                                  const float *__restrict__ er, const float *logits,
                                                                  double slope, int64_t n_rows,
                                                                  GatStat *__restrict__ st, float *alpha,
                                                                  int64_t ahs, int n_long, int64_t long_rows) {
  constexpr int kTile = kStatTileFloats / H;
  constexpr int kRows = kStatWarps * (32 / H);  // rows per short CTA (32 / H per warp)
  __shared__ __align__(16) float s_tile[kStatWarps][kStatTileFloats];
  __shared__ int64_t s_rp[kRows + 1];
  __shared__ uint8_t s_rowof[kApply ? kStatWarps : 1][kApply ? kTile : 1];            // batch row of an entry
  __shared__ __align__(16) float s_invw[kApply ? kStatWarps : 1][kApply ? 32 : 1];   // 1 / S per (batch row, head)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const double slope_l2e = slope * kLog2e;
  float *T = s_tile[warp];
#if GSP_STAT_TRACE
  if (tid == 0 && blockIdx.x < kTraceMax) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_stat_trace[0][blockIdx.x] = gtimer();
    g_stat_trace[2][blockIdx.x] = smid;
    g_stat_trace[3][blockIdx.x] = (int)blockIdx.x < n_long;
  }
  struct TraceEnd {
    int lane;
    __device__ ~TraceEnd() {
      if (lane == 0 && blockIdx.x < kTraceMax) atomicMax(&g_stat_trace[1][blockIdx.x], gtimer());
    }
  } trace_end{(int)(threadIdx.x & 31)};
#endif
  if ((int)blockIdx.x < n_long) {
    constexpr int kSl = LongSlots<H>::kSlots;
    __shared__ double s_pm[kSl][kStatWarps][H], s_ps[kSl][kStatWarps][H], s_M[kSl][H];
    __shared__ float s_inv[kSl][H];
    __shared__ int64_t s_lr[kSl], s_lb[2 * kSl + 1];  // rows; starts [0, kSl), ends at [1 + nk + k]
    __shared__ int s_pre[kSl + 1], s_list[kThreads], s_cnt;
    const int64_t r0 = (int64_t)blockIdx.x * long_rows, r1 = min(n_rows, r0 + long_rows);
    for (int64_t base = r0; base < r1; base += kThreads) {
      if (tid == 0) s_cnt = 0;
      __syncthreads();
      const int64_t r = base + tid;
      if (r < r1 && __ldg(rp + r + 1) - __ldg(rp + r) > kTile) s_list[atomicAdd(&s_cnt, 1)] = tid;
      __syncthreads();
      const int cnt = s_cnt;
      for (int g0 = 0; g0 < cnt; g0 += kSl) {
        const int nk = min(kSl, cnt - g0);
        if (tid == 0) {  // the group's rows, their extents and chunk offsets
          int pre = 0;
          for (int k = 0; k < nk; ++k) {
            const int64_t rr = base + s_list[g0 + k], b = __ldg(rp + rr), e = __ldg(rp + rr + 1);
            s_lr[k] = rr;
            s_lb[k] = b;
            s_lb[1 + nk + k] = e;
            s_pre[k] = pre;
            pre += (int)((e - b + kTile - 1) / kTile);
          }
          s_pre[nk] = pre;
        }
        __syncthreads();
        stat_long_group<H, kScores, kApply>(T, s_pm, s_ps, s_M, s_inv, s_lr, s_lb, s_pre, nk, rp, col, el, er,
                                            logits, slope, slope_l2e, st, alpha, ahs, warp, lane, tid);
      }
      __syncthreads();  // s_list / s_cnt are rewritten
    }
    return;
  }
  const int64_t rbase = (int64_t)(blockIdx.x - n_long) * kRows;
  for (int i = tid; i <= kRows; i += kStatWarps * 32) s_rp[i] = __ldg(rp + min(rbase + i, n_rows));
  __syncthreads();
  stat_short_rows<H, kScores, kApply>(T, s_rowof[kApply ? warp : 0], s_invw[kApply ? warp : 0], s_rp, rbase, n_rows,
                                      col, el, er, logits, slope, st, alpha, ahs, warp, lane);
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
    // long CTAs (a slice of kLongSlice rows each) come first in the grid
    const int64_t long_rows = kLongSlice;
    const int n_long = (int)ceil_div(a->n_rows, long_rows);
    const unsigned blocks = (unsigned)(n_long + ceil_div(a->n_rows, kStatWarps * (32 / H)));
#define GSP_STATS_H(HH)                                                                                       \
  case HH:                                                                                                   \
    row_stats_warp<HH, kScores, kApply><<<blocks, kStatWarps * 32, 0, s>>>(                                   \
        a->row_ptr, a->col_idx, el, er, logits, slope, a->n_rows, st, alpha, ahs, n_long, long_rows);         \
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
    // keep the staged window (col + hpt weight runs) within ~42 KB: smaller
    // row blocks balance better (a 60 KB window measured 0.452 -> 0.477 ms on C3)
    const int hpt = engine_hpt(L, d, heads);
    const int64_t win_max = GSP_HM_WIN_BYTES / (4 * (1 + hpt));
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
