// gat.cu -- GAT path: attention projection (a4), edge softmax (a6) and the
// fused score -> softmax -> multi-head SpMM aggregate (a5+a6+a7).
// PAPER.md P:253 (GAT), P:648-649 (multi-head SpMM), P:653-656 (edge-wise
// softmax with warp-level max / sum reductions); readings A9-A14.
#include "spmm_engine.cuh"

namespace gsp {

// ------------------------------------------------------------------------
// Row statistics: m[u,h] = max_e s[e,h] (fp64) and 1 / sum_e exp(s - m).
// One warp per row; lane l serves head l % H and every (32/H)-th edge, so
// the max and the sum are warp-shuffle reductions over lanes of equal head
// ("warp level intrinsic ... find the max ... reduce ... the sum").
// Order per (row, head): sequential per lane, then an xor tree -> fixed.
// ------------------------------------------------------------------------
// kScores: s from el/er (GAT) or s = logits (edge softmax).
// kApply : write alpha = exp(s - m) / sum in a third pass (standalone edge
//          softmax; logits may alias alpha) instead of storing the statistics.
template <bool kScores, bool kApply>
__global__ void __launch_bounds__(256) row_stats_warp(const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                                                      const float *__restrict__ el, const float *__restrict__ er,
                                                      const float *logits, double slope, int H, int64_t n_rows,
                                                      GatStat *__restrict__ st, float *alpha) {
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= n_rows) return;
  const int lane = threadIdx.x & 31;
  const int h = lane % H, j0 = lane / H, step = 32 / H;
  const int64_t b = __ldg(rp + r), e1 = __ldg(rp + r + 1);
  if (b == e1) return;
  const double el_u = kScores ? (double)__ldg(el + r * H + h) : 0.0;
  auto score = [&](int64_t e) -> double {
    if (kScores) {
      const double t = el_u + (double)__ldg(er + (int64_t)__ldg(col + e) * H + h);
      return t >= 0.0 ? t : slope * t;
    } else {
      return (double)logits[e * H + h];
    }
  };
  double m = -INFINITY;
  for (int64_t e = b + j0; e < e1; e += step) m = fmax(m, score(e));
  for (int off = H; off < 32; off <<= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  double s = 0.0;
  for (int64_t e = b + j0; e < e1; e += step) s += (double)expf((float)(score(e) - m));
  for (int off = H; off < 32; off <<= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (kApply) {
    const float inv_s = (float)(1.0 / s);
    for (int64_t e = b + j0; e < e1; e += step) alpha[e * H + h] = expf((float)(score(e) - m)) * inv_s;
  } else if (lane < H) {
    GatStat g;
    g.m = m;
    g.inv_s = (float)(1.0 / s);
    g.pad = 0.f;
    st[r * H + h] = g;
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
  if (32 % H == 0) {
    const int64_t blocks = ceil_div(a->n_rows, 8);
    row_stats_warp<kScores, kApply><<<(unsigned)blocks, 256, 0, s>>>(a->row_ptr, a->col_idx, el, er, logits, slope,
                                                                      H, a->n_rows, st, alpha);
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
  if (d % 4 == 0 && ldz % 4 == 0 && aligned16(z) && aligned16(a_l) && aligned16(a_r))
    attn_project_warp<4><<<blocks, 256, 0, s>>>(n, heads, d, z, ldz, a_l, a_r, el, er);
  else
    attn_project_warp<1><<<blocks, 256, 0, s>>>(n, heads, d, z, ldz, a_l, a_r, el, er);
  return check_launch("attn_project");
}

extern "C" gsp_status gsp_gat_workspace(const gsp_csr *a, int32_t heads, size_t *ws_bytes) {
  clear_detail();
  if (!a || heads <= 0 || !ws_bytes) return fail(GSP_ERR_INVALID_ARG, "gsp_gat_workspace: bad argument");
  *ws_bytes = 0;  // the softmax statistics live in registers / shared memory of the fused kernel
  return GSP_OK;
}

static gsp_status gat_aggregate_impl(const gsp_csr *a, int32_t heads, const float *el, const float *er,
                                     double negative_slope, const float *z, int64_t d, int64_t ldz, float *y,
                                     int64_t ldy, float *alpha_out, const float *bias, int act, cudaStream_t s,
                                     const char *fn) {
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
  int vmax = 1;
  if (ldz % 4 == 0 && aligned16(z)) vmax = 4;
  else if (ldz % 2 == 0 && aligned8(z)) vmax = 2;
  EngineLaunch L;
  st = engine_plan(a->n_rows, a->n_cols, a->nnz, f, d, vmax, 0, 0, &L, 1);  // one head per team (fp64 state in registers)
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
  p.hpt = engine_hpt(L, d);
  p.bias = bias;
  p.act = act;
  if ((st = engine_ldxv(p, L, a->n_cols, ldz))) return st;
  WeightGat w{el, er, alpha_out, negative_slope, heads};
  return engine_launch(L, p, w, s);
}

extern "C" gsp_status gsp_gat_aggregate(const gsp_csr *a, int32_t heads, const float *el, const float *er,
                                        double negative_slope, const float *z, int64_t d, int64_t ldz, float *y,
                                        int64_t ldy, float *alpha_out, void *ws, size_t ws_bytes, gsp_stream stream) {
  (void)ws;
  (void)ws_bytes;
  return gat_aggregate_impl(a, heads, el, er, negative_slope, z, d, ldz, y, ldy, alpha_out, nullptr, 0, cs(stream),
                            "gsp_gat_aggregate");
}

extern "C" gsp_status gsp_gat_aggregate_bias_act(const gsp_csr *a, int32_t heads, const float *el, const float *er,
                                                 double negative_slope, const float *z, int64_t d, int64_t ldz,
                                                 const float *bias, gsp_act act, float *y, int64_t ldy,
                                                 gsp_stream stream) {
  if (act < GSP_ACT_NONE || act > GSP_ACT_ELU) return fail(GSP_ERR_INVALID_ARG, "gsp_gat_aggregate_bias_act: bad act");
  return gat_aggregate_impl(a, heads, el, er, negative_slope, z, d, ldz, y, ldy, nullptr, bias, (int)act, cs(stream),
                            "gsp_gat_aggregate_bias_act");
}
