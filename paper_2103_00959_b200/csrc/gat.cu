// gat.cu -- GAT path: attention projection (a4), edge softmax (a6) and the
// fused score -> softmax -> multi-head SpMM aggregate (a5+a6+a7).
// PAPER.md P:253 (GAT), P:648-649 (multi-head SpMM), P:653-656 (edge-wise
// softmax with warp-level max / sum reductions); readings A9-A14.
#include "spmm_engine.cuh"

namespace gsp {

// ------------------------------------------------------------------------
// Row statistics: m[u,h] = max_e s[e,h] (fp64) and 1 / sum_e exp(s - m),
// all heads of a row at once ("warp level intrinsic ... find the max
// ... reduce ... the sum").  H (heads, dividing 32) is a template parameter.
// Grid: one CTA of 8 warps per 32 rows; warp w owns rows 4w .. 4w+3 of them.
//  * SHORT rows (<= kTile = 1024 / H entries): the entries of the warp's 4
//    rows (contiguous in CSR) are loaded into the warp's shared tile
//    T[kTile][H] in one sweep when they fit (else row by row); each lane
//    issues all of its loads before the first use (kU entries in flight).
//    Then, per row, lane l reduces head h = l % H over the row's entries
//    part, part + P, ... (part = l / H, P = 32 / H) and an xor tree over
//    lanes of equal head finishes the max and the sum.  exp(s - m) stays in
//    the tile for the apply pass.
//  * LONG rows: the whole CTA, after the short rows.  Warp w takes the
//    tile-sized chunks w, w+8, ... of the row (same tile and lane layout),
//    then the xor tree per warp and the 8 warps' partials in warp order.
// Every order depends on the row alone (deterministic, partition-invariant).
// ------------------------------------------------------------------------
// kScores: s from el/er (GAT) or s = logits (edge softmax).
// kApply : write alpha = exp(s - m) / sum (standalone edge softmax; logits
//          may alias alpha) instead of storing the statistics.
#ifndef GSP_STAT_WARPS
#define GSP_STAT_WARPS 8
#endif
#ifndef GSP_STAT_RPW
#define GSP_STAT_RPW 4
#endif
#ifndef GSP_STAT_MINB
#define GSP_STAT_MINB 4
#endif
constexpr int kStatWarps = GSP_STAT_WARPS;  // warps per CTA
constexpr int kStatRPW = GSP_STAT_RPW;      // rows per warp
constexpr int kStatTileFloats = 1024;  // per warp: kTile = 1024 / H entries x H heads (4 KB)

template <bool kScores>
__device__ __forceinline__ double stat_score(float t, double el_u, double slope) {
  if (kScores) {
    const double x = el_u + (double)t;
    return x >= 0.0 ? x : slope * x;
  }
  return (double)t;
}

// entries [e0, e0 + cnt) of the CSR -> T[j][H] (er rows of their columns, or logits rows)
template <int H, bool kScores>
__device__ __forceinline__ void stat_load(float *T, int64_t e0, int cnt, const int32_t *__restrict__ col,
                                          const float *__restrict__ er, const float *logits, int lane) {
  if (kScores) {
    constexpr int kU = (32 / H) < 4 ? ((32 / H) < 1 ? 1 : 32 / H) : 4;  // entries per lane per round
    constexpr int kV = H >= 4 ? 4 : H;                                 // floats per load
    using VT = typename VecT<kV>::T;
    for (int base = 0; base < cnt; base += 32 * kU) {
      int c[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int j = base + lane + 32 * u;
        c[u] = j < cnt ? __ldg(col + e0 + j) : 0;
      }
      float v[kU][H];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int j = base + lane + 32 * u;
#pragma unroll
        for (int q = 0; q < H; q += kV) {
          if (j < cnt) {
            float t[kV];
            vld<kV>(t, reinterpret_cast<const VT *>(er + (int64_t)c[u] * H + q));
#pragma unroll
            for (int i = 0; i < kV; ++i) v[u][q + i] = t[i];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int j = base + lane + 32 * u;
        if (j < cnt) {
#pragma unroll
          for (int q = 0; q < H; q += kV) {
            float t[kV];
#pragma unroll
            for (int i = 0; i < kV; ++i) t[i] = v[u][q + i];
            Vec<kV>::st_shared(T + j * H + q, t);
          }
        }
      }
    }
  } else {
    const float *src = logits + e0 * H;  // cnt rows of H logits are contiguous
    const int nf = cnt * H;
    constexpr int kU = 8;
    for (int base = 0; base < nf; base += 32 * kU) {
      float v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int k = base + lane + 32 * u;
        v[u] = k < nf ? src[k] : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int k = base + lane + 32 * u;
        if (k < nf) T[k] = v[u];
      }
    }
  }
}

// reduce one short row held in T[0 .. d) and write its statistics or alpha
template <int H, bool kScores, bool kApply>
__device__ __forceinline__ void stat_row(float *T, int64_t r, int64_t b, int d, const float *__restrict__ el,
                                         double slope, GatStat *__restrict__ st, float *alpha, int lane) {
  constexpr int P = 32 / H;
  const int h = lane % H, part = lane / H;
  const double el_u = kScores ? (double)__ldg(el + r * H + h) : 0.0;
  // the score is monotone non-decreasing in the stored value (LeakyReLU with
  // slope >= 0 and IEEE RN are monotone), so the row max of the fp64 scores is
  // the score of the fp32 max -- exactly (slope < 0: fp64 max of the scores)
  float mr = -INFINITY;
  for (int j = part; j < d; j += P) mr = fmaxf(mr, T[j * H + h]);
#pragma unroll
  for (int off = H; off < 32; off <<= 1) mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, off));
  double m = stat_score<kScores>(mr, el_u, slope);
  if (kScores && !(slope >= 0.0)) {
    m = -INFINITY;
    for (int j = part; j < d; j += P) m = fmax(m, stat_score<kScores>(T[j * H + h], el_u, slope));
#pragma unroll
    for (int off = H; off < 32; off <<= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  }
  double s = 0.0;
  for (int j = part; j < d; j += P) {
    const float ex = expf((float)(stat_score<kScores>(T[j * H + h], el_u, slope) - m));
    s += (double)ex;
    if (kApply) T[j * H + h] = ex;  // own slot: no other lane reads it
  }
#pragma unroll
  for (int off = H; off < 32; off <<= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  const float inv_s = (float)(1.0 / s);
  if (kApply) {
    for (int j = part; j < d; j += P) alpha[(b + j) * H + h] = T[j * H + h] * inv_s;  // lane-contiguous
  } else if (part == 0) {
    GatStat g;
    g.m = m;
    g.inv_s = inv_s;
    g.pad = 0.f;
    st[r * H + h] = g;
  }
}

template <int H, bool kScores, bool kApply>
__global__ void __launch_bounds__(kStatWarps * 32, GSP_STAT_MINB) row_stats_warp(const int64_t *__restrict__ rp,
                                                                  const int32_t *__restrict__ col,
                                                                  const float *__restrict__ el,
                                                                  const float *__restrict__ er, const float *logits,
                                                                  double slope, int64_t n_rows,
                                                                  GatStat *__restrict__ st, float *alpha) {
  constexpr int kTile = kStatTileFloats / H;
  __shared__ __align__(16) float s_tile[kStatWarps][kStatTileFloats];
  __shared__ int s_long[kStatWarps * kStatRPW];
  __shared__ int s_nlong;
  __shared__ double s_red[kStatWarps][H];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  if (tid == 0) s_nlong = 0;
  __syncthreads();
  const int64_t rbase = (int64_t)blockIdx.x * kStatWarps * kStatRPW;
  {
    float *T = s_tile[warp];
    const int64_t r0 = rbase + warp * kStatRPW;
    const int64_t bl = (lane <= kStatRPW) ? __ldg(rp + min(r0 + lane, n_rows)) : 0;
    int64_t B[kStatRPW + 1];
#pragma unroll
    for (int k = 0; k <= kStatRPW; ++k) B[k] = __shfl_sync(0xffffffffu, bl, k);
    const bool together = B[kStatRPW] - B[0] <= kTile;
    if (together) stat_load<H, kScores>(T, B[0], (int)(B[kStatRPW] - B[0]), col, er, logits, lane);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kStatRPW; ++k) {
      const int64_t d = B[k + 1] - B[k];
      if (d == 0) continue;
      if (d > kTile) {
        if (lane == 0) s_long[atomicAdd(&s_nlong, 1)] = warp * kStatRPW + k;
        continue;
      }
      float *Tk = T;
      if (together) {
        Tk = T + (B[k] - B[0]) * H;
      } else {
        __syncwarp();
        stat_load<H, kScores>(T, B[k], (int)d, col, er, logits, lane);
        __syncwarp();
      }
      stat_row<H, kScores, kApply>(Tk, r0 + k, B[k], (int)d, el, slope, st, alpha, lane);
    }
  }
  __syncthreads();
  // long rows: the whole CTA; warp w takes tile-sized chunks w, w+8, ... of
  // the row (same tile loads and lane layout as short rows), partials of the
  // 8 warps combined in warp order
  const int nlong = s_nlong;
  float *T = s_tile[warp];
  constexpr int P = 32 / H;
  const int h = lane % H, part = lane / H;
  for (int k = 0; k < nlong; ++k) {
    const int64_t r = rbase + s_long[k];
    const int64_t b = __ldg(rp + r), e1 = __ldg(rp + r + 1);
    const double el_u = kScores ? (double)__ldg(el + r * H + h) : 0.0;
    const bool resident = (e1 - b) <= (int64_t)kStatWarps * kTile;  // one chunk per warp: no reloads
    double m = -INFINITY, sum = 0.0;
    for (int pass = 0; pass < (kApply ? 3 : 2); ++pass) {
      const float inv_s = pass == 2 ? (float)(1.0 / sum) : 0.0f;
      double acc = pass == 0 ? -INFINITY : 0.0;
      for (int64_t c0 = b + (int64_t)warp * kTile; c0 < e1; c0 += (int64_t)kStatWarps * kTile) {
        const int cnt = (int)min((int64_t)kTile, e1 - c0);
        if (pass == 0 || !resident) {  // a row of <= 8 tiles keeps each warp's chunk in its tile
          __syncwarp();
          stat_load<H, kScores>(T, c0, cnt, col, er, logits, lane);
          __syncwarp();
        }
        if (pass == 0) {  // max of the stored values, then of the scores (monotone, see stat_row)
          float mr = -INFINITY;
          for (int j = part; j < cnt; j += P) mr = fmaxf(mr, T[j * H + h]);
          if (mr != -INFINITY) acc = fmax(acc, stat_score<kScores>(mr, el_u, slope));
          if (kScores && !(slope >= 0.0))
            for (int j = part; j < cnt; j += P) acc = fmax(acc, stat_score<kScores>(T[j * H + h], el_u, slope));
          continue;
        }
        for (int j = part; j < cnt; j += P) {
          const double sc = stat_score<kScores>(T[j * H + h], el_u, slope);
          if (pass == 1) acc += (double)expf((float)(sc - m));
          else alpha[(c0 + j) * H + h] = expf((float)(sc - m)) * inv_s;
        }
      }
      if (pass == 2) break;
#pragma unroll
      for (int off = H; off < 32; off <<= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, acc, off);
        acc = pass == 0 ? fmax(acc, o) : acc + o;
      }
      if (part == 0) s_red[warp][h] = acc;
      __syncthreads();
      double x = s_red[0][h];
      for (int w = 1; w < kStatWarps; ++w) x = pass == 0 ? fmax(x, s_red[w][h]) : x + s_red[w][h];
      __syncthreads();
      if (pass == 0) m = x;
      else sum = x;
    }
    if (!kApply && warp == 0 && part == 0) {
      GatStat g;
      g.m = m;
      g.inv_s = (float)(1.0 / sum);
      g.pad = 0.f;
      st[r * H + h] = g;
    }
  }
}

// Fallback for H not dividing 32: one thread per (row, head), sequential.
template <bool kScores, bool kApply>
__global__ void row_stats_thread(const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                                 const float *__restrict__ el, const float *__restrict__ er, const float *logits,
                                 double slope, int H, int64_t n_rows, GatStat *__restrict__ st, float *alpha) {
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
    for (int64_t e = b; e < e1; ++e) alpha[e * H + h] = expf((float)(score(e) - m)) * inv_s;
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
                               int H, GatStat *st, float *alpha, cudaStream_t s) {
  if (a->n_rows == 0) return GSP_OK;
  const float *vsrc = kScores ? er : logits;
  const bool vec_ok = H < 4 ? (H == 1 || aligned8(vsrc)) : aligned16(vsrc);
  if (32 % H == 0 && (vec_ok || !kScores)) {
    const unsigned blocks = (unsigned)ceil_div(a->n_rows, kStatWarps * kStatRPW);
#define GSP_STATS_H(HH)                                                                                       \
  case HH:                                                                                                   \
    row_stats_warp<HH, kScores, kApply><<<blocks, kStatWarps * 32, 0, s>>>(a->row_ptr, a->col_idx, el, er,     \
                                                                         logits, slope, a->n_rows, st, alpha); \
    break;
    switch (H) {
      GSP_STATS_H(1) GSP_STATS_H(2) GSP_STATS_H(4) GSP_STATS_H(8) GSP_STATS_H(16) GSP_STATS_H(32)
    }
#undef GSP_STATS_H
  } else {
    const int64_t blocks = ceil_div(a->n_rows * H, 256);
    row_stats_thread<kScores, kApply><<<(unsigned)blocks, 256, 0, s>>>(a->row_ptr, a->col_idx, el, er, logits,
                                                                        slope, H, a->n_rows, st, alpha);
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

extern "C" gsp_status gsp_gat_workspace(const gsp_csr *a, int32_t heads, size_t *ws_bytes) {
  clear_detail();
  if (!a || heads <= 0 || !ws_bytes) return fail(GSP_ERR_INVALID_ARG, "gsp_gat_workspace: bad argument");
  *ws_bytes = (size_t)std::max<int64_t>(a->n_rows, 0) * heads * sizeof(GatStat);  // (m, 1/S) per (row, head)
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
  const size_t need = (size_t)a->n_rows * heads * sizeof(GatStat);
  const bool pre = ws && ws_bytes >= need && aligned16(ws) && 32 % heads == 0;
  EngineLaunch L;
  st = engine_plan(a->n_rows, a->n_cols, a->nnz, f, d, vmax, 0, 0, &L, pre ? kMaxHpt : 1);
  if (st) return st;
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
