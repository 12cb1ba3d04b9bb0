// backward.cu -- NEXT-3: the GAT backward operators.  PAPER.md P:652 (§4.1:
// SDDMM T = A (.) (P Q^T) "is used for back-propagating the gradients to the
// sparse adjacency matrix since the adjacency matrix of the GAT model is
// computed by the attention mechanism"); edge softmax P:653-656.
//
//   gsp_csr_transpose        A^T (canonical) + perm: entry e' of A^T is entry
//                            perm[e'] of A (radix sort of column keys)
//   gsp_sddmm                out[e,h] = <p[u,h,:], q[v,h,:]>, e = (u,v)
//   gsp_edge_softmax_backward ds = alpha (dalpha - sum_row alpha dalpha)
//   gsp_gat_aggregate_backward  dZ, d_el, d_er of the fused GAT aggregate
//   gsp_attn_project_backward   dZ += d_el a_l + d_er a_r; d_al, d_ar
#include <algorithm>

#include "spmm_engine.cuh"

namespace gsp {

// radix helpers from build.cu
gsp_status radix_sort_pairs(uint64_t *&keys, uint32_t *&vals, uint64_t *keys_alt, uint32_t *vals_alt, int64_t N,
                            int bits, uint32_t *counts, uint8_t *scan_ws, cudaStream_t s);
size_t radix_counts_bytes(int64_t N);
size_t radix_scan_ws_bytes(int64_t N);

static size_t a256(size_t b) { return (b + 255) & ~size_t(255); }

// ------------------------------------------------------------------ transpose
__global__ void transpose_keys_kernel(const int32_t *__restrict__ col, int64_t nnz, uint64_t *__restrict__ keys,
                                      uint32_t *__restrict__ vals) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    keys[e] = (uint64_t)(uint32_t)col[e];
    vals[e] = (uint32_t)e;
  }
}

__global__ void row_of_kernel(const int64_t *__restrict__ rp, int64_t n, int32_t *__restrict__ row_of) {
  const int64_t u = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (u >= n) return;
  for (int64_t e = rp[u] + (threadIdx.x & 31); e < rp[u + 1]; e += 32) row_of[e] = (int32_t)u;
}

// col_t[k] = row of entry perm[k]; row_ptr_t from the sorted column keys
__global__ void transpose_finish_kernel(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ perm,
                                        int64_t nnz, int64_t n_cols, const int32_t *__restrict__ row_of,
                                        int64_t *__restrict__ rp_t, int32_t *__restrict__ col_t,
                                        int32_t *__restrict__ perm_out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t e = perm[k];
    col_t[k] = row_of[e];
    perm_out[k] = (int32_t)e;
    const int64_t c = (int64_t)keys[k];
    const int64_t prev = k == 0 ? -1 : (int64_t)keys[k - 1];
    for (int64_t cc = prev + 1; cc <= c; ++cc) rp_t[cc] = k;  // columns that start here (gap fill)
    if (k == nnz - 1)
      for (int64_t cc = c + 1; cc <= n_cols; ++cc) rp_t[cc] = nnz;
  }
}

__global__ void fill_i64(int64_t *p, int64_t count, int64_t v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

struct TransposeLayout {
  size_t ka, kb, va, vb, counts, scan, row_of, total;
};
static TransposeLayout transpose_layout(int64_t nnz) {
  TransposeLayout L{};
  size_t off = 0;
  auto take = [&](size_t b) {
    const size_t o = off;
    off += a256(std::max<size_t>(b, 1));
    return o;
  };
  L.ka = take((size_t)nnz * 8);
  L.kb = take((size_t)nnz * 8);
  L.va = take((size_t)nnz * 4);
  L.vb = take((size_t)nnz * 4);
  L.counts = take(radix_counts_bytes(nnz));
  L.scan = take(radix_scan_ws_bytes(nnz));
  L.row_of = take((size_t)nnz * 4);
  L.total = off;
  return L;
}

// ---------------------------------------------------------------------- SDDMM
// Each warp owns 64 consecutive entries (edge-balanced, hub rows split across
// warps); the row of the first entry comes from a warp-cooperative search.
// Lane l holds float4 column slices l*4 + 128k of p[u]; per edge and head the
// dot product is the lane's fma chain over its 4 columns, then an xor tree
// over the D/4 lanes of that head (fixed order).
constexpr int kSddmmEdgesPerWarp = 64;
constexpr int kSddmmMaxChunks = 8;  // H*D <= 1024 on the vector path

// H heads of width D starting at column 0 of p / q; out[e * Hout + h0 + h]
template <int NC>  // 128-float chunks of the H*D row per lane group (NC * 128 >= H*D)
__global__ void __launch_bounds__(256) sddmm_vec_kernel(const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                                                        int64_t n, int64_t nnz, int H, int D,
                                                        const float *__restrict__ p, int64_t ldp,
                                                        const float *__restrict__ q, int64_t ldq,
                                                        float *__restrict__ out, int Hout, int h0) {
  constexpr int U = NC >= 8 ? 1 : 8 / NC;  // edges whose q rows are in flight together
  static_assert(kSddmmEdgesPerWarp == 64, "two column indices per lane");
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int64_t e0 = warp * kSddmmEdgesPerWarp;
  if (e0 >= nnz) return;
  const int64_t e1 = min(nnz, e0 + kSddmmEdgesPerWarp);
  // the warp's column indices, loaded once (coalesced) and broadcast by shuffle
  const int cl0 = e0 + lane < e1 ? __ldg(col + e0 + lane) : 0;
  const int cl1 = e0 + 32 + lane < e1 ? __ldg(col + e0 + 32 + lane) : 0;
  // u = the row holding entry e0: first r with rp[r] > e0, minus one
  int64_t u = warp_lower_bound(rp, n, e0 + 1) - 1;
  int64_t u_end = __ldg(rp + u + 1);
  const int W = H * D, lpg = D / 4;  // lanes per head group
  float4 pv[NC];
  auto load_p = [&]() {
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int c = 4 * lane + 128 * k;
      pv[k] = c < W ? __ldg(reinterpret_cast<const float4 *>(p + u * ldp + c)) : make_float4(0, 0, 0, 0);
    }
  };
  load_p();
  for (int64_t eb = e0; eb < e1; eb += U) {
    float4 qv[U][NC];
#pragma unroll
    for (int t = 0; t < U; ++t) {  // every q gather of the batch before the first use
      const int i = (int)(eb - e0) + t;
      const int v0 = __shfl_sync(0xffffffffu, cl0, i & 31), v1 = __shfl_sync(0xffffffffu, cl1, i & 31);
      const int64_t v = i < 32 ? v0 : v1;
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        const int c = 4 * lane + 128 * k;
        qv[t][k] = (eb + t < e1 && c < W) ? __ldg(reinterpret_cast<const float4 *>(q + v * ldq + c))
                                          : make_float4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int t = 0; t < U; ++t) {
      const int64_t e = eb + t;
      if (e >= e1) break;
      while (e >= u_end) {  // next row (warp-uniform)
        ++u;
        u_end = __ldg(rp + u + 1);
        load_p();
      }
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        const int c = 4 * lane + 128 * k;
        float acc = 0.0f;
        acc = fmaf(pv[k].x, qv[t][k].x, acc);
        acc = fmaf(pv[k].y, qv[t][k].y, acc);
        acc = fmaf(pv[k].z, qv[t][k].z, acc);
        acc = fmaf(pv[k].w, qv[t][k].w, acc);
        for (int o = 1; o < lpg; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (c < W && (lane % lpg) == 0) out[e * Hout + h0 + c / D] = acc;
      }
    }
  }
}

// Transposed reduction (LPG = D/4 lanes per head, LPG <= 16): a batch of up to
// LPG consecutive entries of ONE row is gathered together; each lane forms
// its 4-column partial dot for every entry of the batch, then a butterfly
// reduce-scatter over the head's LPG lanes (LPG-1 shuffles instead of
// LPG*log2(LPG)) leaves the full dot of entry j in the head's lane j.
// Order per (entry, head): lane fma chain over x,y,z,w, then the butterfly
// from distance LPG/2 down to 1 -- fixed.
template <int LPG, int NC>
__global__ void __launch_bounds__(256, 2) sddmm_tr_kernel(const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                                                          int64_t n, int64_t nnz, int H, int D,
                                                          const float *__restrict__ p, int64_t ldp,
                                                          const float *__restrict__ q, int64_t ldq,
                                                          float *__restrict__ out) {
  static_assert(kSddmmEdgesPerWarp == 64, "two column indices per lane");
  const int lane = threadIdx.x & 31, gl = lane % LPG;
  const int64_t warp = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int64_t e0 = warp * kSddmmEdgesPerWarp;
  if (e0 >= nnz) return;
  const int64_t e1 = min(nnz, e0 + kSddmmEdgesPerWarp);
  const int cl0 = e0 + lane < e1 ? __ldg(col + e0 + lane) : 0;
  const int cl1 = e0 + 32 + lane < e1 ? __ldg(col + e0 + 32 + lane) : 0;
  int64_t u = warp_lower_bound(rp, n, e0 + 1) - 1;
  int64_t u_end = __ldg(rp + u + 1);
  const int W = H * D;
  float4 pv[NC];
  auto load_p = [&]() {
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int c = 4 * lane + 128 * k;
      pv[k] = c < W ? __ldg(reinterpret_cast<const float4 *>(p + u * ldp + c)) : make_float4(0, 0, 0, 0);
    }
  };
  load_p();
  int64_t e = e0;
  while (e < e1) {
    while (e >= u_end) {  // next row (warp-uniform)
      ++u;
      u_end = __ldg(rp + u + 1);
      load_p();
    }
    const int cnt = (int)min((int64_t)LPG, min(u_end, e1) - e);
    int vcol[LPG];
#pragma unroll
    for (int i = 0; i < LPG; ++i) {
      const int idx = (int)(e - e0) + i;
      const int a0 = __shfl_sync(0xffffffffu, cl0, idx & 31), a1 = __shfl_sync(0xffffffffu, cl1, idx & 31);
      vcol[i] = idx < 32 ? a0 : a1;
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int c = 4 * lane + 128 * k;
      float4 qv[LPG];
#pragma unroll
      for (int i = 0; i < LPG; ++i)  // every gather of the batch before the first use
        qv[i] = (i < cnt && c < W) ? __ldg(reinterpret_cast<const float4 *>(q + (int64_t)vcol[i] * ldq + c))
                                   : make_float4(0, 0, 0, 0);
      float v[LPG];
#pragma unroll
      for (int i = 0; i < LPG; ++i) {
        float acc = 0.0f;
        acc = fmaf(pv[k].x, qv[i].x, acc);
        acc = fmaf(pv[k].y, qv[i].y, acc);
        acc = fmaf(pv[k].z, qv[i].z, acc);
        acc = fmaf(pv[k].w, qv[i].w, acc);
        v[i] = acc;
      }
#pragma unroll
      for (int m = LPG / 2; m >= 1; m >>= 1) {  // reduce-scatter: lane j of the group ends with entry j
        const bool hi = (lane & m) != 0;
#pragma unroll
        for (int i = 0; i < m; ++i) {
          const float send = hi ? v[i] : v[i + m];
          const float keep = hi ? v[i + m] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
        }
      }
      const int cg = 128 * k + 4 * (lane - gl);  // first column of this lane's head group
      if (gl < cnt && cg < W) out[(e + gl) * H + cg / D] = v[0];
    }
    e += cnt;
  }
}

// generic path: one thread per (entry, head), sequential dot product
__global__ void sddmm_scalar_kernel(const int64_t *__restrict__ rp, const int32_t *__restrict__ col, int64_t n,
                                    int64_t nnz, int H, int D, const float *__restrict__ p, int64_t ldp,
                                    const float *__restrict__ q, int64_t ldq, float *__restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nnz * H; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / H;
    const int h = (int)(t % H);
    int64_t lo = 0, hi = n;  // row of e: last r with rp[r] <= e
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) / 2;
      if (rp[mid] <= e) lo = mid; else hi = mid;
    }
    const float *pu = p + lo * ldp + (int64_t)h * D, *qv = q + (int64_t)col[e] * ldq + (int64_t)h * D;
    float acc = 0.0f;
    for (int k = 0; k < D; ++k) acc = fmaf(pu[k], qv[k], acc);
    out[t] = acc;
  }
}

// ------------------------------------------------------ softmax backward (+GAT)
// One warp per row; lane l serves head l % H and every (32/H)-th entry.
// kGat: also dt = ds * leaky'(el[u] + er[v]) written over ds, d_el = row sum.
template <bool kGat>
__global__ void __launch_bounds__(256) softmax_bwd_warp(const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                                                        int64_t n, int H, const float *__restrict__ alpha,
                                                        const float *dalpha, float *ds, const float *__restrict__ el,
                                                        const float *__restrict__ er, double slope,
                                                        float *__restrict__ d_el) {
  // one warp per row; rows longer than kSbLong entries: the whole CTA after
  // its short rows (threads t take entries t/H + k*256/H, head t%H; partials
  // xor-reduced per warp, then the 8 warps in order) -- a single warp would
  // walk a hub row sequentially
  constexpr int kSbLong = 256;
  __shared__ int s_long[8];
  __shared__ int s_nlong;
  __shared__ double s_red[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_nlong = 0;
  __syncthreads();
  auto row_pass = [&](int64_t r, int64_t b, int64_t e1, int t, int nthreads, bool cta) {
    const int h = t % H, j0 = t / H, step = nthreads / H;
    double dot = 0.0;
#pragma unroll 4
    for (int64_t e = b + j0; e < e1; e += step) dot += (double)alpha[e * H + h] * (double)dalpha[e * H + h];
    for (int off = H; off < 32; off <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
    if (cta) {
      if (lane < H) s_red[warp][lane] = dot;
      __syncthreads();
      dot = s_red[0][h];
      for (int w = 1; w < 8; ++w) dot += s_red[w][h];
      __syncthreads();
    }
    double rs = 0.0;
    const double el_u = kGat ? (double)__ldg(el + r * H + h) : 0.0;
    for (int64_t e0 = b + j0; e0 < e1; e0 += 4 * (int64_t)step) {
      // 4 entries' loads before their stores (ds may alias dalpha entry-wise)
      float a4[4], d4[4], t4[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t e = e0 + k * (int64_t)step;
        a4[k] = e < e1 ? alpha[e * H + h] : 0.0f;
        d4[k] = e < e1 ? dalpha[e * H + h] : 0.0f;
        t4[k] = (kGat && e < e1) ? __ldg(er + (int64_t)__ldg(col + e) * H + h) : 0.0f;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t e = e0 + k * (int64_t)step;
        if (e < e1) {
          double g = (double)a4[k] * ((double)d4[k] - dot);
          if (kGat) {
            const double tt = el_u + (double)t4[k];
            g = tt >= 0.0 ? g : g * slope;
            rs += g;
          }
          ds[e * H + h] = (float)g;
        }
      }
    }
    if (kGat) {
      for (int off = H; off < 32; off <<= 1) rs += __shfl_xor_sync(0xffffffffu, rs, off);
      if (cta) {
        if (lane < H) s_red[warp][lane] = rs;
        __syncthreads();
        rs = s_red[0][h];
        for (int w = 1; w < 8; ++w) rs += s_red[w][h];
        __syncthreads();
        if (threadIdx.x < H) d_el[r * H + h] = (float)rs;
      } else if (lane < H) {
        d_el[r * H + h] = (float)rs;
      }
    }
  };
  const int64_t r = (int64_t)blockIdx.x * 8 + warp;
  if (r < n) {
    const int64_t b = __ldg(rp + r), e1 = __ldg(rp + r + 1);
    if (e1 - b > kSbLong) {
      if (lane == 0) s_long[atomicAdd(&s_nlong, 1)] = warp;
    } else if (e1 > b) {
      row_pass(r, b, e1, lane, 32, false);
    } else if (kGat && lane < H) {
      d_el[r * H + lane] = 0.0f;
    }
  }
  __syncthreads();
  for (int k = 0; k < s_nlong; ++k) {
    const int64_t rr = (int64_t)blockIdx.x * 8 + s_long[k];
    row_pass(rr, __ldg(rp + rr), __ldg(rp + rr + 1), threadIdx.x, 256, true);
  }
}

// column sums through the transpose: out[v,h] = sum_{e' in row v of A^T} vals[perm[e'], h]
__global__ void __launch_bounds__(256) colsum_warp(const int64_t *__restrict__ rpt, const int32_t *__restrict__ perm,
                                                   int64_t n_cols, int H, const float *__restrict__ vals,
                                                   float *__restrict__ out) {
  // one warp per column; columns with more than 256 entries: the whole CTA
  // after its short columns (partials xor-reduced per warp, warps in order)
  __shared__ int s_long[8];
  __shared__ int s_nlong;
  __shared__ double s_red[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_nlong = 0;
  __syncthreads();
  auto col_sum = [&](int64_t v, int t, int nthreads) {
    const int h = t % H, j0 = t / H, step = nthreads / H;
    double s = 0.0;
    const int64_t kend = __ldg(rpt + v + 1);
#pragma unroll 4
    for (int64_t k = __ldg(rpt + v) + j0; k < kend; k += step) s += (double)vals[(int64_t)__ldg(perm + k) * H + h];
    for (int off = H; off < 32; off <<= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    return s;
  };
  const int64_t v = (int64_t)blockIdx.x * 8 + warp;
  if (v < n_cols) {
    if (__ldg(rpt + v + 1) - __ldg(rpt + v) > 256) {
      if (lane == 0) s_long[atomicAdd(&s_nlong, 1)] = warp;
    } else {
      const double s = col_sum(v, lane, 32);
      if (lane < H) out[v * H + lane] = (float)s;
    }
  }
  __syncthreads();
  for (int k = 0; k < s_nlong; ++k) {
    const int64_t vv = (int64_t)blockIdx.x * 8 + s_long[k];
    const double s = col_sum(vv, threadIdx.x, 256);
    if (lane < H) s_red[warp][lane] = s;
    __syncthreads();
    if (threadIdx.x < H) {
      double t = s_red[0][threadIdx.x];
      for (int w = 1; w < 8; ++w) t += s_red[w][threadIdx.x];
      out[vv * H + threadIdx.x] = (float)t;
    }
    __syncthreads();
  }
}

// ----------------------------------------------------- attn projection backward
// dz[u,h,:] += d_el[u,h] a_l[h,:] + d_er[u,h] a_r[h,:]   (one thread per element)
__global__ void attn_bwd_dz_kernel(int64_t n, int H, int D, const float *__restrict__ d_el,
                                   const float *__restrict__ d_er, const float *__restrict__ al,
                                   const float *__restrict__ ar, float *__restrict__ dz, int64_t lddz) {
  const int64_t W = (int64_t)H * D;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * W; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = t / W;
    const int k = (int)(t % W), h = k / D;
    float v = dz[u * lddz + k];
    v = fmaf(d_el[u * H + h], al[k], v);
    v = fmaf(d_er[u * H + h], ar[k], v);
    dz[u * lddz + k] = v;
  }
}
// d_al[k] = sum_u d_el[u,h] z[u,k] (k in head h): per-block partials over a
// fixed row range, then a fixed-order final sum -> deterministic.
constexpr int kAttnRowsPerBlock = 256;
__global__ void attn_bwd_partial_kernel(int64_t n, int H, int D, const float *__restrict__ d_el,
                                        const float *__restrict__ d_er, const float *__restrict__ z, int64_t ldz,
                                        double *__restrict__ part /*[nblk][2W]*/) {
  const int64_t W = (int64_t)H * D;
  const int64_t u0 = (int64_t)blockIdx.x * kAttnRowsPerBlock, u1 = min(n, u0 + kAttnRowsPerBlock);
  for (int64_t k = threadIdx.x; k < W; k += blockDim.x) {
    const int h = (int)(k / D);
    double sl = 0.0, sr = 0.0;
    for (int64_t u = u0; u < u1; ++u) {
      const double zv = (double)z[u * ldz + k];
      sl += (double)d_el[u * H + h] * zv;
      sr += (double)d_er[u * H + h] * zv;
    }
    part[(int64_t)blockIdx.x * 2 * W + k] = sl;
    part[(int64_t)blockIdx.x * 2 * W + W + k] = sr;
  }
}
__global__ void attn_bwd_final_kernel(int64_t nblk, int64_t W, const double *__restrict__ part,
                                      float *__restrict__ d_al, float *__restrict__ d_ar) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < 2 * W; k += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t b = 0; b < nblk; ++b) s += part[b * 2 * W + k];
    if (k < W) d_al[k] = (float)s;
    else d_ar[k - W] = (float)s;
  }
}

// weight functor for the transposed multi-head SpMM: alpha of the original entry
struct WeightAlphaPerm {
  const float *alpha;
  const int32_t *perm;
  int heads;
  struct Row {
    static constexpr bool kUnit = false, kComputed = false, kStagedVal = false, kMultiHead = true, kInStats = false;
    const float *alpha;
    const int32_t *perm;
    int heads, h;
    __device__ __forceinline__ float w(int64_t e, int, int hh) const {
      return __ldg(alpha + (int64_t)__ldg(perm + e) * heads + h + hh);
    }
  };
  __device__ __forceinline__ Row row(int64_t, int h, bool, void *) const { return Row{alpha, perm, heads, h}; }
};

static gsp_status launch_sddmm(const gsp_csr *a, int H, int64_t D, const float *p, int64_t ldp, const float *q,
                               int64_t ldq, float *out, cudaStream_t s) {
  if (a->nnz == 0) return GSP_OK;
  const int64_t W = H * D;
  const bool vec = D % 4 == 0 && D / 4 <= 32 && ((D / 4) & (D / 4 - 1)) == 0 && W <= 128 * kSddmmMaxChunks &&
                   ldp % 4 == 0 && ldq % 4 == 0 && aligned16(p) && aligned16(q);
  if (vec) {
    const int64_t warps = ceil_div(a->nnz, kSddmmEdgesPerWarp);
    const unsigned gb = (unsigned)ceil_div(warps, 8);
    const int lpg = (int)(D / 4), nc = (int)((W + 127) / 128);
    if (lpg >= 2 && lpg <= 16 && nc <= 4) {
#define GSP_SDDMM_TR(L, NCV)                                                                                 \
  sddmm_tr_kernel<L, NCV><<<gb, 256, 0, s>>>(a->row_ptr, a->col_idx, a->n_rows, a->nnz, H, (int)D, p, ldp, q, ldq, out)
#define GSP_SDDMM_TR_NC(L)        \
  if (nc <= 1) GSP_SDDMM_TR(L, 1); \
  else if (nc <= 2) GSP_SDDMM_TR(L, 2); \
  else GSP_SDDMM_TR(L, 4);
      switch (lpg) {
        case 2: GSP_SDDMM_TR_NC(2) break;
        case 4: GSP_SDDMM_TR_NC(4) break;
        case 8: GSP_SDDMM_TR_NC(8) break;
        case 16: GSP_SDDMM_TR_NC(16) break;
      }
#undef GSP_SDDMM_TR_NC
#undef GSP_SDDMM_TR
    } else {  // (128-column slab launches measured slower on C3: 1.35 vs 1.23 ms)
#define GSP_SDDMM_NC(NCV)                                                                                       \
  sddmm_vec_kernel<NCV><<<gb, 256, 0, s>>>(a->row_ptr, a->col_idx, a->n_rows, a->nnz, H, (int)D, p, ldp, q, ldq, out, \
                                           H, 0)
      if (nc <= 1) GSP_SDDMM_NC(1);
      else if (nc <= 2) GSP_SDDMM_NC(2);
      else if (nc <= 4) GSP_SDDMM_NC(4);
      else GSP_SDDMM_NC(8);
#undef GSP_SDDMM_NC
    }
  } else {
    sddmm_scalar_kernel<<<(unsigned)std::min<int64_t>(ceil_div(a->nnz * H, 256), 65535 * 8), 256, 0, s>>>(
        a->row_ptr, a->col_idx, a->n_rows, a->nnz, H, (int)D, p, ldp, q, ldq, out);
  }
  return check_launch("sddmm");
}

}  // namespace gsp

using namespace gsp;

extern "C" gsp_status gsp_csr_transpose_workspace(const gsp_csr *a, size_t *ws_bytes) {
  clear_detail();
  if (!a || !ws_bytes || a->nnz < 0) return fail(GSP_ERR_INVALID_ARG, "gsp_csr_transpose_workspace: bad argument");
  *ws_bytes = transpose_layout(a->nnz).total;
  return GSP_OK;
}

extern "C" gsp_status gsp_csr_transpose(const gsp_csr *a, int64_t *row_ptr_t, int32_t *col_t, int32_t *perm,
                                        void *ws, size_t ws_bytes, gsp_stream stream) {
  const char *fn = "gsp_csr_transpose";
  clear_detail();
  gsp_status st = check_csr(a, false, fn);
  if (st) return st;
  if (a->nnz >= (int64_t(1) << 31)) return fail(GSP_ERR_UNSUPPORTED, "%s: nnz must be < 2^31", fn);
  if (!row_ptr_t || (a->nnz > 0 && (!col_t || !perm))) return fail(GSP_ERR_INVALID_ARG, "%s: null output", fn);
  const TransposeLayout L = transpose_layout(a->nnz);
  if (!ws || ws_bytes < L.total) return fail(GSP_ERR_WORKSPACE, "%s: workspace needs %zu bytes", fn, L.total);
  if (reinterpret_cast<uintptr_t>(ws) & 255u) return fail(GSP_ERR_WORKSPACE, "%s: ws must be 256-byte aligned", fn);
  cudaStream_t s = cs(stream);
  if (a->nnz == 0) {
    fill_i64<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(a->n_cols + 1, 256), 4096)), 256, 0, s>>>(
        row_ptr_t, a->n_cols + 1, 0);
    return check_launch("transpose(empty)");
  }
  uint8_t *W = reinterpret_cast<uint8_t *>(ws);
  uint64_t *ka = reinterpret_cast<uint64_t *>(W + L.ka), *kb = reinterpret_cast<uint64_t *>(W + L.kb);
  uint32_t *va = reinterpret_cast<uint32_t *>(W + L.va), *vb = reinterpret_cast<uint32_t *>(W + L.vb);
  int32_t *row_of = reinterpret_cast<int32_t *>(W + L.row_of);
  const unsigned gb = (unsigned)std::min<int64_t>(ceil_div(a->nnz, 256), 65535 * 4);
  transpose_keys_kernel<<<gb, 256, 0, s>>>(a->col_idx, a->nnz, ka, va);
  if ((st = check_launch("transpose_keys"))) return st;
  row_of_kernel<<<(unsigned)ceil_div(a->n_rows, 8), 256, 0, s>>>(a->row_ptr, a->n_rows, row_of);
  if ((st = check_launch("row_of"))) return st;
  int bits = 1;
  while (bits < 40 && (int64_t(1) << bits) <= a->n_cols) ++bits;
  if ((st = radix_sort_pairs(ka, va, kb, vb, a->nnz, bits, reinterpret_cast<uint32_t *>(W + L.counts), W + L.scan,
                             s)))
    return st;
  fill_i64<<<1, 32, 0, s>>>(row_ptr_t, 1, 0);
  transpose_finish_kernel<<<gb, 256, 0, s>>>(ka, va, a->nnz, a->n_cols, row_of, row_ptr_t, col_t, perm);
  return check_launch("transpose_finish");
}

extern "C" gsp_status gsp_sddmm(const gsp_csr *a, int32_t heads, const float *p, int64_t d, int64_t ldp,
                                const float *q, int64_t ldq, float *out, gsp_stream stream) {
  const char *fn = "gsp_sddmm";
  clear_detail();
  gsp_status st = check_csr(a, false, fn);
  if (st) return st;
  if (heads <= 0 || d < 0 || ldp < heads * d || ldq < heads * d)
    return fail(GSP_ERR_INVALID_ARG, "%s: need heads >= 1, ldp, ldq >= heads*d", fn);
  if (a->nnz == 0) return GSP_OK;
  if (!p || !q || !out) return fail(GSP_ERR_INVALID_ARG, "%s: null pointer", fn);
  return launch_sddmm(a, heads, d, p, ldp, q, ldq, out, cs(stream));
}

extern "C" gsp_status gsp_edge_softmax_backward(const gsp_csr *a, int32_t heads, const float *alpha,
                                                const float *dalpha, float *ds, gsp_stream stream) {
  const char *fn = "gsp_edge_softmax_backward";
  clear_detail();
  gsp_status st = check_csr(a, false, fn);
  if (st) return st;
  if (heads <= 0 || 32 % heads) return fail(GSP_ERR_UNSUPPORTED, "%s: heads must divide 32", fn);
  if (a->nnz == 0 || a->n_rows == 0) return GSP_OK;
  if (!alpha || !dalpha || !ds) return fail(GSP_ERR_INVALID_ARG, "%s: null pointer", fn);
  softmax_bwd_warp<false><<<(unsigned)ceil_div(a->n_rows, 8), 256, 0, cs(stream)>>>(
      a->row_ptr, a->col_idx, a->n_rows, heads, alpha, dalpha, ds, nullptr, nullptr, 0.0, nullptr);
  return check_launch("softmax_bwd");
}

extern "C" gsp_status gsp_gat_backward_workspace(const gsp_csr *a, int32_t heads, size_t *ws_bytes) {
  clear_detail();
  if (!a || heads <= 0 || !ws_bytes) return fail(GSP_ERR_INVALID_ARG, "gsp_gat_backward_workspace: bad argument");
  *ws_bytes = 2 * a256((size_t)std::max<int64_t>(a->nnz, 1) * heads * 4);
  return GSP_OK;
}

extern "C" gsp_status gsp_gat_aggregate_backward(const gsp_csr *a, const gsp_csr *at, const int32_t *perm,
                                                 int32_t heads, const float *el, const float *er,
                                                 double negative_slope, const float *z, int64_t d, int64_t ldz,
                                                 const float *dy, int64_t lddy, float *dz, int64_t lddz, float *d_el,
                                                 float *d_er, void *ws, size_t ws_bytes, gsp_stream stream) {
  const char *fn = "gsp_gat_aggregate_backward";
  clear_detail();
  gsp_status st = check_csr(a, false, fn);
  if (st || (st = check_csr(at, false, fn))) return st;
  const int64_t f = (int64_t)heads * d;
  if (heads <= 0 || 32 % heads) return fail(GSP_ERR_UNSUPPORTED, "%s: heads must divide 32", fn);
  if (d < 0 || ldz < f || lddy < f || lddz < f) return fail(GSP_ERR_INVALID_ARG, "%s: bad leading dimensions", fn);
  if (a->n_rows != a->n_cols || at->n_rows != a->n_cols || at->n_cols != a->n_rows || at->nnz != a->nnz)
    return fail(GSP_ERR_INVALID_ARG, "%s: at must be the transpose of a square a", fn);
  if (a->n_rows == 0) return GSP_OK;
  if (!el || !er || !z || !dy || !dz || !d_el || !d_er || (a->nnz && !perm))
    return fail(GSP_ERR_INVALID_ARG, "%s: null pointer", fn);
  size_t need = 0;
  gsp_gat_backward_workspace(a, heads, &need);
  if (!ws || ws_bytes < need) return fail(GSP_ERR_WORKSPACE, "%s: workspace needs %zu bytes", fn, need);
  cudaStream_t s = cs(stream);
  if (validate_mode()) {  // the score inputs el / er must be finite
    const float *arr[2] = {el, er};
    const int64_t cnt[2] = {a->n_rows * heads, a->n_cols * heads};
    const char *nm[2] = {"el", "er"};
    if ((st = check_finite(s, fn, 2, arr, cnt, nm))) return st;
  }
  float *alpha = reinterpret_cast<float *>(ws);
  float *g = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(ws) + a256((size_t)std::max<int64_t>(a->nnz, 1) *
                                                                                 heads * 4));
  // 1. alpha = softmax_row(LeakyReLU(el[u] + er[v]))  (same kernel as gsp_gat_aggregate's statistics)
  if ((st = launch_row_softmax_scores(a, el, er, negative_slope, heads, alpha, s))) return st;
  // 2. dalpha = SDDMM(dy, z)
  if ((st = launch_sddmm(a, heads, d, dy, lddy, z, ldz, g, s))) return st;
  // 3. dt = (alpha (dalpha - <alpha, dalpha>)) * leaky'(t) in place; d_el = row sums
  softmax_bwd_warp<true><<<(unsigned)ceil_div(a->n_rows, 8), 256, 0, s>>>(
      a->row_ptr, a->col_idx, a->n_rows, heads, alpha, g, g, el, er, negative_slope, d_el);
  if ((st = check_launch("gat softmax_bwd"))) return st;
  // 4. d_er = column sums of dt (through the transpose)
  colsum_warp<<<(unsigned)ceil_div(at->n_rows, 8), 256, 0, s>>>(at->row_ptr, perm, at->n_rows, heads, g, d_er);
  if ((st = check_launch("colsum"))) return st;
  // 5. dz = A^T-weighted multi-head SpMM of dy with alpha[perm]
  if (f == 0) return GSP_OK;
  int vmax = 1;
  if (lddy % 4 == 0 && aligned16(dy)) vmax = 4;
  else if (lddy % 2 == 0 && aligned8(dy)) vmax = 2;
  EngineLaunch L;
  if ((st = engine_plan(at->n_rows, at->n_cols, at->nnz, f, d, vmax, 0, 0, &L, kMaxHpt))) return st;
  EngineParams p;
  p.row_ptr = at->row_ptr;
  p.col = at->col_idx;
  p.x = dy;
  p.y = dz;
  p.n_rows = at->n_rows;
  p.ldx = lddy;
  p.ldy = lddz;
  p.f = f;
  p.block_nnz = L.block_nnz;
  p.nblk = L.nblk;
  p.head_dim = d;
  p.y_vec_ok = engine_y_vec_ok(L, dz, lddz);
  engine_stage(p, L, at->nnz, at->col_idx, nullptr);
  p.hpt = engine_hpt(L, d, heads);
  if ((st = engine_ldxv(p, L, at->n_cols, lddy))) return st;
  return engine_launch(L, p, WeightAlphaPerm{alpha, perm, heads}, s);
}

extern "C" gsp_status gsp_attn_project_backward_workspace(int64_t n, int32_t heads, int64_t d, size_t *ws_bytes) {
  clear_detail();
  if (n < 0 || heads <= 0 || d < 0 || !ws_bytes) return fail(GSP_ERR_INVALID_ARG, "bad argument");
  *ws_bytes = (size_t)std::max<int64_t>(1, ceil_div(n, kAttnRowsPerBlock)) * 2 * heads * d * 8;
  return GSP_OK;
}

extern "C" gsp_status gsp_attn_project_backward(int64_t n, int32_t heads, int64_t d, const float *z, int64_t ldz,
                                                const float *a_l, const float *a_r, const float *d_el,
                                                const float *d_er, float *dz, int64_t lddz, float *d_al, float *d_ar,
                                                void *ws, size_t ws_bytes, gsp_stream stream) {
  const char *fn = "gsp_attn_project_backward";
  clear_detail();
  const int64_t W = (int64_t)heads * d;
  if (n < 0 || heads <= 0 || d < 0 || ldz < W || lddz < W) return fail(GSP_ERR_INVALID_ARG, "%s: bad sizes", fn);
  if (n == 0 || W == 0) return GSP_OK;
  if (!z || !a_l || !a_r || !d_el || !d_er || !dz || !d_al || !d_ar)
    return fail(GSP_ERR_INVALID_ARG, "%s: null pointer", fn);
  size_t need = 0;
  gsp_attn_project_backward_workspace(n, heads, d, &need);
  if (!ws || ws_bytes < need) return fail(GSP_ERR_WORKSPACE, "%s: workspace needs %zu bytes", fn, need);
  cudaStream_t s = cs(stream);
  const int64_t nblk = ceil_div(n, kAttnRowsPerBlock);
  attn_bwd_partial_kernel<<<(unsigned)nblk, 256, 0, s>>>(n, heads, (int)d, d_el, d_er, z, ldz,
                                                         reinterpret_cast<double *>(ws));
  gsp_status st = check_launch("attn_bwd_partial");
  if (st) return st;
  attn_bwd_final_kernel<<<(unsigned)ceil_div(2 * W, 256), 256, 0, s>>>(nblk, W, reinterpret_cast<double *>(ws), d_al,
                                                                       d_ar);
  if ((st = check_launch("attn_bwd_final"))) return st;
  attn_bwd_dz_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n * W, 256), 65535 * 8), 256, 0, s>>>(
      n, heads, (int)d, d_el, d_er, a_l, a_r, dz, lddz);
  return check_launch("attn_bwd_dz");
}
