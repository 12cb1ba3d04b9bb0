// spmm.cu -- gsp_spmm / gsp_spmm_ex / gsp_multihead_spmm (§4.1,
// Eq. formula:1 P:640-645; multi-head SpMM P:648-649).
#include "spmm_engine.cuh"

namespace gsp {

static int64_t pow2_floor(int64_t v) {
  int64_t p = 1;
  while (p * 2 <= v) p *= 2;
  return p;
}

// L2 bytes we aim to keep one slab of X in (126 MB L2; leave room for the
// streamed CSR, Y and the next slab).  DESIGN.md §Kernels / slab sizing.
static constexpr int64_t kL2SlabBudget = 48ll << 20;

gsp_status engine_plan(int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t f, int64_t head_dim, int vmax,
                       int32_t slab_req, int32_t block_req, EngineLaunch *L, int max_hpt) {
  int V = vmax;
  int64_t SW = 0;
  if (head_dim > 0 && head_dim == f && slab_req <= 0) head_dim = 0;  // one head cannot be straddled: plain plan
  if (head_dim > 0) {
    while (V > 1 && head_dim % V) V /= 2;
    const int64_t heads = f / head_dim;
    if (slab_req > 0) {
      SW = slab_req;
      const bool whole = SW % head_dim == 0 && (SW / head_dim) <= kMaxHpt && heads % (SW / head_dim) == 0;
      if (SW % V || SW / V > 32 || (SW / V & (SW / V - 1)) || !(head_dim % SW == 0 || whole))
        return fail(GSP_ERR_INVALID_ARG, "slab_cols %d must divide head_dim %lld or be up to %d whole heads",
                    slab_req, (long long)head_dim, kMaxHpt);
    } else {
      // prefer a slab of hpt whole heads (hpt | heads, hpt <= kMaxHpt, <= 128 columns); else slabs inside a head
      SW = 0;
      for (int64_t hpt = std::min<int64_t>(max_hpt, heads); hpt >= 1 && !SW; --hpt) {
        const int64_t sw = hpt * head_dim, g = sw / V;
        if (heads % hpt == 0 && sw <= 128 && sw % V == 0 && g >= 1 && g <= 32 && (g & (g - 1)) == 0) SW = sw;
      }
      if (!SW) {
        int64_t G = 32;
        while (G > 1 && (head_dim % (G * V) || G * V > 128)) G /= 2;
        SW = G * V;
      }
    }
  } else {
    if (slab_req > 0) {
      SW = slab_req;
      if (SW == 256 && V == 4) {
        V = 8;  // two float4 per lane
      } else if (SW % V || SW / V > 32 || (SW / V & (SW / V - 1))) {
        return fail(GSP_ERR_INVALID_ARG, "slab_cols %d must be V*2^k with k<=5 (V=%d) or 256", slab_req, V);
      }
    } else {
      // widest single-float4-per-lane slab (measured best on C4, DESIGN.md
      // §Slab sizing); the L2-resident width is kept for reference
      (void)kL2SlabBudget;
      (void)pow2_floor;
      SW = 32 * V;
      // no slab wider than the (vector-rounded) feature width
      int64_t fw = ((f + V - 1) / V) * V;
      while (SW / 2 >= fw && SW / 2 >= V) SW /= 2;
    }
  }
  L->V = V;
  L->G = (int)(SW / V);
  L->slab_cols = SW;
  L->nslab = ceil_div(f, SW);
  const int64_t T = L->G >= 8 ? 32 : 4 * L->G;  // team size (see Team<G>)
  int64_t C = block_req > 0 ? block_req : std::min<int64_t>(8192, (kThreads / T) * 512);
  if (block_req <= 0) {
    // keep >= ~8 CTAs per SM over the whole grid for small graphs
    const int64_t want = 8ll * sm_count();
    const int64_t cap = (nnz * L->nslab) / want;
    if (cap < C) C = std::max<int64_t>(256, cap);
  }
  C = std::min<int64_t>(C, (int64_t)kHub * (kMaxHubPerBlock - 1));
  C = std::max<int64_t>(C, 1);
  L->block_nnz = C;
  L->nblk = nnz / C + 1;
  (void)n_rows;
  return GSP_OK;
}

// The slab plan of one gsp_spmm call: the main launch covers [0, f_main) with
// slab width L.slab_cols; when the last slab would leave more than half of its
// lanes idle, the remaining columns [f_main, f) go to a second, narrower launch.
struct SpmmPlan {
  EngineLaunch main, tail;
  int64_t f_main, f_tail;
};

static gsp_status spmm_plan(const gsp_csr *a, const float *x, int64_t f, int64_t ldx, const gsp_spmm_opts *opts,
                            SpmmPlan *P) {
  int vmax = 1;
  if (ldx % 4 == 0 && aligned16(x)) vmax = 4;
  else if (ldx % 2 == 0 && aligned8(x)) vmax = 2;
  const int32_t slab_req = opts ? opts->slab_cols : 0, block_req = opts ? opts->block_nnz : 0;
  // 256-column slabs read two float4 per lane (32 bytes): the last vector of a
  // row must stay inside [0, ldx), so ldx % 8 == 0 and a 32-byte aligned base
  if (slab_req == 256 && vmax == 4 && !(ldx % 8 == 0 && reinterpret_cast<uintptr_t>(x) % 32 == 0))
    return fail(GSP_ERR_INVALID_ARG, "slab_cols 256 needs ldx %% 8 == 0 and a 32-byte aligned x");
  gsp_status st = engine_plan(a->n_rows, a->n_cols, a->nnz, f, 0, vmax, slab_req, block_req, &P->main, 1);
  if (st) return st;
  P->f_main = f;
  P->f_tail = 0;
  const int64_t SW = P->main.slab_cols, rem = f % SW;
  if (slab_req == 0 && P->main.V == 4 && f > SW && rem && rem <= SW / 2) {
    int64_t tw = 16;
    while (tw < rem) tw *= 2;
    st = engine_plan(a->n_rows, a->n_cols, a->nnz, rem, 0, vmax, (int32_t)tw, block_req, &P->tail, 1);
    if (st) return st;
    P->f_main = f - rem;
    P->f_tail = rem;
    P->main.nslab = P->f_main / SW;
  }
  return GSP_OK;
}

// accumulate epilogue of a propagation step (see gsp_spmm_accumulate)
struct AccEpi {
  float *acc;
  int64_t ldacc;
  float coef;
  const float *src;
  int64_t ldsrc;
  float src_coef;
};

static gsp_status spmm_launch_part(const gsp_csr *a, const EngineLaunch &L, const float *x, int64_t f, int64_t ldx,
                                   float *y, int64_t ldy, gsp_reduce red, const AccEpi *epi, cudaStream_t s,
                                   const float *bias = nullptr, int act = 0) {
  EngineParams p;
  p.row_ptr = a->row_ptr;
  p.col = a->col_idx;
  p.x = x;
  p.y = y;
  p.n_rows = a->n_rows;
  p.ldx = ldx;
  p.ldy = ldy;
  p.f = f;
  p.block_nnz = L.block_nnz;
  p.nblk = L.nblk;
  p.head_dim = 0;
  p.y_vec_ok = engine_y_vec_ok(L, y, ldy);
  engine_stage(p, L, a->nnz, a->col_idx, a->val);
  p.bias = bias;
  p.act = act;
  if (epi) {
    const int vw = L.V == 8 ? 4 : L.V;
    p.acc = epi->acc;
    p.ldacc = epi->ldacc;
    p.acc_coef = epi->coef;
    p.acc_src = epi->src;
    p.ldsrc = epi->ldsrc;
    p.src_coef = epi->src_coef;
    p.skip_y = y == nullptr;
    p.acc_vec_ok = (epi->ldacc % vw == 0) && (reinterpret_cast<uintptr_t>(epi->acc) % (4 * vw) == 0);
    p.src_vec_ok = epi->src && (epi->ldsrc % vw == 0) && (reinterpret_cast<uintptr_t>(epi->src) % (4 * vw) == 0);
    if (!y) p.y = epi->acc;  // never written (skip_y); keeps pointer arithmetic valid
  }
  gsp_status st = engine_ldxv(p, L, a->n_cols, ldx);
  if (st) return st;
  p.mean = red == GSP_REDUCE_MEAN;
  switch (red) {
    case GSP_REDUCE_SUM:
    case GSP_REDUCE_MEAN:
      return a->val ? engine_launch(L, p, WeightVal{a->val}, s) : engine_launch(L, p, WeightOne{}, s);
    case GSP_REDUCE_MAX:
      return a->val ? engine_launch<WeightVal, RedMax>(L, p, WeightVal{a->val}, s)
                    : engine_launch<WeightOne, RedMax>(L, p, WeightOne{}, s);
    case GSP_REDUCE_MIN:
      return a->val ? engine_launch<WeightVal, RedMin>(L, p, WeightVal{a->val}, s)
                    : engine_launch<WeightOne, RedMin>(L, p, WeightOne{}, s);
  }
  return fail(GSP_ERR_INVALID_ARG, "bad reduce op %d", (int)red);
}

static gsp_status spmm_impl(const gsp_csr *a, const float *x, int64_t f, int64_t ldx, float *y, int64_t ldy,
                            const gsp_spmm_opts *opts, gsp_reduce red, cudaStream_t s, const char *fn) {
  clear_detail();
  if (red < GSP_REDUCE_SUM || red > GSP_REDUCE_MIN) return fail(GSP_ERR_INVALID_ARG, "%s: bad reduce op", fn);
  gsp_status st = check_csr(a, false, fn);
  if (st) return st;
  if (f < 0 || ldx < f || ldy < f) return fail(GSP_ERR_INVALID_ARG, "%s: need f >= 0, ldx >= f, ldy >= f", fn);
  if (a->n_rows == 0 || f == 0) return GSP_OK;
  if (!y) return fail(GSP_ERR_INVALID_ARG, "%s: y is NULL", fn);
  if (a->n_cols > 0 && !x) return fail(GSP_ERR_INVALID_ARG, "%s: x is NULL", fn);
  const size_t xb = a->n_cols ? (size_t)((a->n_cols - 1) * ldx + f) * 4 : 0;
  const size_t yb = (size_t)((a->n_rows - 1) * ldy + f) * 4;
  if (overlaps(x, xb, y, yb)) return fail(GSP_ERR_ALIAS, "%s: x and y overlap", fn);
  SpmmPlan P;
  if ((st = spmm_plan(a, x, f, ldx, opts, &P))) return st;
  if ((st = spmm_launch_part(a, P.main, x, P.f_main, ldx, y, ldy, red, nullptr, s))) return st;
  if (P.f_tail) st = spmm_launch_part(a, P.tail, x + P.f_main, P.f_tail, ldx, y + P.f_main, ldy, red, nullptr, s);
  return st;
}

static gsp_status spmm_acc_impl(const gsp_csr *a, const float *x, int64_t f, int64_t ldx, float *t, int64_t ldt,
                                float *acc, int64_t ldacc, float coef, const float *src, int64_t ldsrc, float src_coef,
                                cudaStream_t s, const char *fn) {
  gsp_status st = check_csr(a, false, fn);
  if (st) return st;
  if (f < 0 || ldx < f || (t && ldt < f) || ldacc < f || (src && ldsrc < f))
    return fail(GSP_ERR_INVALID_ARG, "%s: bad f / leading dimensions", fn);
  if (a->n_rows == 0 || f == 0) return GSP_OK;
  if (!x || !acc) return fail(GSP_ERR_INVALID_ARG, "%s: x / acc is NULL", fn);
  const size_t xb = a->n_cols ? (size_t)((a->n_cols - 1) * ldx + f) * 4 : 0;
  const size_t ab = (size_t)((a->n_rows - 1) * ldacc + f) * 4;
  const size_t tb = t ? (size_t)((a->n_rows - 1) * ldt + f) * 4 : 0;
  if (overlaps(x, xb, acc, ab) || (t && (overlaps(x, xb, t, tb) || overlaps(t, tb, acc, ab))))
    return fail(GSP_ERR_ALIAS, "%s: x, t and acc must not overlap", fn);
  if (src && src != acc && overlaps(src, (size_t)((a->n_rows - 1) * ldsrc + f) * 4, acc, ab))
    return fail(GSP_ERR_ALIAS, "%s: src partially overlaps acc", fn);
  SpmmPlan P;
  if ((st = spmm_plan(a, x, f, ldx, nullptr, &P))) return st;
  AccEpi e{acc, ldacc, coef, src, ldsrc, src_coef};
  if ((st = spmm_launch_part(a, P.main, x, P.f_main, ldx, t, t ? ldt : 0, GSP_REDUCE_SUM, &e, s))) return st;
  if (P.f_tail) {
    AccEpi e2{acc + P.f_main, ldacc, coef, src ? src + P.f_main : nullptr, ldsrc, src_coef};
    st = spmm_launch_part(a, P.tail, x + P.f_main, P.f_tail, ldx, t ? t + P.f_main : nullptr, t ? ldt : 0,
                          GSP_REDUCE_SUM, &e2, s);
  }
  return st;
}

}  // namespace gsp

using namespace gsp;

extern "C" gsp_status gsp_spmm(const gsp_csr *a, const float *x, int64_t f, int64_t ldx, float *y, int64_t ldy,
                               gsp_stream stream) {
  return spmm_impl(a, x, f, ldx, y, ldy, nullptr, GSP_REDUCE_SUM, cs(stream), "gsp_spmm");
}

// fp16 feature storage (P:1302-1320 mixed precision): y (fp32) = A x with x in
// fp16, products and sums in fp32.  Same engine, order and epilogue as
// gsp_spmm; V = 4 halves (8-byte gathers, 128-column slabs: half of fp32's
// L2 footprint per slab) when ldx % 4 == 0 and x is 8-byte aligned, else
// scalar halves (V = 8, 16-byte gathers, is available via GSP_F16_VMAX=8).
static gsp_status spmm_f16_part(const gsp_csr *a, const EngineLaunch &L, const __half *x, int64_t f, int64_t ldx,
                                float *y, int64_t ldy, cudaStream_t s) {
  EngineParams p;
  p.row_ptr = a->row_ptr;
  p.col = a->col_idx;
  p.x = x;
  p.y = y;
  p.n_rows = a->n_rows;
  p.ldx = ldx;
  p.ldy = ldy;
  p.f = f;
  p.block_nnz = L.block_nnz;
  p.nblk = L.nblk;
  p.head_dim = 0;
  p.y_vec_ok = engine_y_vec_ok(L, y, ldy);
  engine_stage(p, L, a->nnz, a->col_idx, a->val);
  const int64_t ldxv = ldx / L.V;  // in 16-byte (V = 8) or 2-byte (V = 1) units
  if (a->n_cols > 0 && (a->n_cols - 1) * ldxv + ldxv >= (int64_t(1) << 32))
    return fail(GSP_ERR_UNSUPPORTED, "feature matrix too large for 32-bit vector offsets");
  p.ldxv = (uint32_t)ldxv;
  return a->val ? engine_launch_f16(L, p, WeightVal{a->val}, s) : engine_launch_f16(L, p, WeightOne{}, s);
}

extern "C" gsp_status gsp_spmm_f16(const gsp_csr *a, const void *x, int64_t f, int64_t ldx, float *y, int64_t ldy,
                                   gsp_stream stream) {
  const char *fn = "gsp_spmm_f16";
  clear_detail();
  gsp_status st = check_csr(a, false, fn);
  if (st) return st;
  if (f < 0 || ldx < f || ldy < f) return fail(GSP_ERR_INVALID_ARG, "%s: need f >= 0, ldx >= f, ldy >= f", fn);
  if (a->n_rows == 0 || f == 0) return GSP_OK;
  if (!y) return fail(GSP_ERR_INVALID_ARG, "%s: y is NULL", fn);
  if (a->n_cols > 0 && !x) return fail(GSP_ERR_INVALID_ARG, "%s: x is NULL", fn);
  const size_t xbytes = a->n_cols ? (size_t)((a->n_cols - 1) * ldx + f) * 2 : 0;
  const size_t ybytes = (size_t)((a->n_rows - 1) * ldy + f) * 4;
  if (overlaps(x, xbytes, y, ybytes)) return fail(GSP_ERR_ALIAS, "%s: x and y overlap", fn);
#ifndef GSP_F16_VMAX
#define GSP_F16_VMAX 4  // measured (tools/f16_probe.py): 4 halves per lane (128-column slabs, 60 MB of X per
                        // slab on C4) 3.9 ms vs 8 halves (256 columns, 2 CTAs/SM) 4.7 ms; fp32 5.4 ms
#endif
  int vmax = 1;
  if (GSP_F16_VMAX >= 8 && ldx % 8 == 0 && aligned16(x)) vmax = 8;
  else if (ldx % 4 == 0 && aligned8(x)) vmax = 4;
  EngineLaunch L, T;
#ifndef GSP_F16_SLAB
#define GSP_F16_SLAB 0  // 0: the engine's default (32 lanes x V)
#endif
  const int32_t slab_req = (GSP_F16_SLAB > 0 && vmax == 4 && f > GSP_F16_SLAB) ? GSP_F16_SLAB : 0;
  if ((st = engine_plan(a->n_rows, a->n_cols, a->nnz, f, 0, vmax, slab_req, 0, &L, 1))) return st;
  const __half *xh = static_cast<const __half *>(x);
  const int64_t SW = L.slab_cols, rem = f % SW;
  cudaStream_t s = cs(stream);
  if (L.V >= 4 && f > SW && rem && rem <= SW / 2) {  // narrower tail launch (as gsp_spmm)
    int64_t tw = 16;
    while (tw < rem) tw *= 2;
    if ((st = engine_plan(a->n_rows, a->n_cols, a->nnz, rem, 0, vmax, (int32_t)tw, 0, &T, 1))) return st;
    L.nslab = (f - rem) / SW;
    if ((st = spmm_f16_part(a, L, xh, f - rem, ldx, y, ldy, s))) return st;
    return spmm_f16_part(a, T, xh + (f - rem), rem, ldx, y + (f - rem), ldy, s);
  }
  return spmm_f16_part(a, L, xh, f, ldx, y, ldy, s);
}

extern "C" gsp_status gsp_spmm_blocked(const gsp_csr *blocks, int32_t nblocks, const float *x, int64_t f, int64_t ldx,
                                       float *y, int64_t ldy, gsp_stream stream) {
  const char *fn = "gsp_spmm_blocked";
  clear_detail();
  if (!blocks || nblocks < 1) return fail(GSP_ERR_INVALID_ARG, "%s: nblocks >= 1 blocks required", fn);
  for (int k = 0; k < nblocks; ++k) {
    gsp_status st = check_csr(&blocks[k], false, fn);
    if (st) return st;
    if (blocks[k].n_rows != blocks[0].n_rows || blocks[k].n_cols != blocks[0].n_cols)
      return fail(GSP_ERR_INVALID_ARG, "%s: blocks must share n_rows and n_cols", fn);
  }
  cudaStream_t s = cs(stream);
  // block 0 writes y, every further block adds its partial once (fixed order)
  gsp_status st = spmm_impl(&blocks[0], x, f, ldx, y, ldy, nullptr, GSP_REDUCE_SUM, s, fn);
  for (int k = 1; k < nblocks && !st; ++k)
    st = spmm_acc_impl(&blocks[k], x, f, ldx, nullptr, 0, y, ldy, 1.0f, nullptr, 0, 0.0f, s, fn);
  return st;
}

extern "C" gsp_status gsp_spmm_accumulate(const gsp_csr *a, const float *x, int64_t f, int64_t ldx, float *t,
                                          int64_t ldt, float *acc, int64_t ldacc, float coef, const float *src,
                                          int64_t ldsrc, float src_coef, gsp_stream stream) {
  clear_detail();
  return spmm_acc_impl(a, x, f, ldx, t, ldt, acc, ldacc, coef, src, ldsrc, src_coef, cs(stream),
                       "gsp_spmm_accumulate");
}

extern "C" gsp_status gsp_propagate_workspace(const gsp_csr *a, int64_t f, int64_t K, size_t *ws_bytes) {
  clear_detail();
  if (!a || f < 0 || K < 0 || !ws_bytes) return fail(GSP_ERR_INVALID_ARG, "gsp_propagate_workspace: bad argument");
  const int64_t ld = (f + 3) / 4 * 4;
  *ws_bytes = K >= 2 ? (size_t)(K >= 3 ? 2 : 1) * (size_t)a->n_rows * ld * 4 + 512 : 0;
  return GSP_OK;
}

extern "C" gsp_status gsp_propagate(const gsp_csr *a, const float *x, int64_t f, int64_t ldx, int64_t K,
                                    const double *theta, float *y, int64_t ldy, void *ws, size_t ws_bytes,
                                    gsp_stream stream) {
  const char *fn = "gsp_propagate";
  clear_detail();
  gsp_status st = check_csr(a, false, fn);
  if (st) return st;
  if (K < 0 || !theta) return fail(GSP_ERR_INVALID_ARG, "%s: K >= 0 and theta[K+1] required", fn);
  if (a->n_rows != a->n_cols) return fail(GSP_ERR_INVALID_ARG, "%s: propagation needs a square matrix", fn);
  if (f < 0 || ldx < f || ldy < f) return fail(GSP_ERR_INVALID_ARG, "%s: bad f / leading dimensions", fn);
  if (a->n_rows == 0 || f == 0) return GSP_OK;
  if (!x || !y) return fail(GSP_ERR_INVALID_ARG, "%s: x / y is NULL", fn);
  size_t need = 0;
  gsp_propagate_workspace(a, f, K, &need);
  if (need && (!ws || ws_bytes < need)) return fail(GSP_ERR_WORKSPACE, "%s: workspace needs %zu bytes", fn, need);
  cudaStream_t s = cs(stream);
  const int64_t ld = (f + 3) / 4 * 4;
  float *tb[2] = {nullptr, nullptr};
  if (need) {
    float *w = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
    tb[0] = w;
    tb[1] = K >= 3 ? w + (size_t)a->n_rows * ld : nullptr;
  }
  if (K == 0) {  // y = theta_0 x: a propagation of zero steps is an epilogue-only pass
    return fail(GSP_ERR_UNSUPPORTED, "%s: K == 0 (y = theta_0 x) is a plain scale; use K >= 1", fn);
  }
  // step k: t_k = A t_{k-1} (t_0 = x); y = theta_k t_k + (k == 1 ? theta_0 x : y)
  const float *tin = x;
  int64_t ldin = ldx;
  for (int64_t k = 1; k <= K; ++k) {
    float *tout = (k == K) ? nullptr : tb[(k - 1) & 1];
    st = spmm_acc_impl(a, tin, f, ldin, tout, ld, y, ldy, (float)theta[k], k == 1 ? x : nullptr, ldx,
                       (float)theta[0], s, fn);
    if (st) return st;
    tin = tout;
    ldin = ld;
  }
  return GSP_OK;
}

extern "C" gsp_status gsp_spmm_bias_act(const gsp_csr *a, const float *x, int64_t f, int64_t ldx, const float *bias,
                                        gsp_act act, float *y, int64_t ldy, gsp_stream stream) {
  const char *fn = "gsp_spmm_bias_act";
  clear_detail();
  if (act < GSP_ACT_NONE || act > GSP_ACT_ELU) return fail(GSP_ERR_INVALID_ARG, "%s: bad activation", fn);
  gsp_status st = check_csr(a, false, fn);
  if (st) return st;
  if (f < 0 || ldx < f || ldy < f) return fail(GSP_ERR_INVALID_ARG, "%s: need f >= 0, ldx >= f, ldy >= f", fn);
  if (a->n_rows == 0 || f == 0) return GSP_OK;
  if (!y || (a->n_cols > 0 && !x)) return fail(GSP_ERR_INVALID_ARG, "%s: null pointer", fn);
  const size_t xb = a->n_cols ? (size_t)((a->n_cols - 1) * ldx + f) * 4 : 0;
  if (overlaps(x, xb, y, (size_t)((a->n_rows - 1) * ldy + f) * 4)) return fail(GSP_ERR_ALIAS, "%s: x and y overlap", fn);
  SpmmPlan P;
  if ((st = spmm_plan(a, x, f, ldx, nullptr, &P))) return st;
  cudaStream_t s = cs(stream);
  if ((st = spmm_launch_part(a, P.main, x, P.f_main, ldx, y, ldy, GSP_REDUCE_SUM, nullptr, s, bias, act))) return st;
  if (P.f_tail)
    st = spmm_launch_part(a, P.tail, x + P.f_main, P.f_tail, ldx, y + P.f_main, ldy, GSP_REDUCE_SUM, nullptr, s,
                          bias ? bias + P.f_main : nullptr, act);
  return st;
}

extern "C" gsp_status gsp_gspmm(const gsp_csr *a, gsp_reduce reduce, const float *x, int64_t f, int64_t ldx, float *y,
                                int64_t ldy, gsp_stream stream) {
  return spmm_impl(a, x, f, ldx, y, ldy, nullptr, reduce, cs(stream), "gsp_gspmm");
}

extern "C" gsp_status gsp_spmm_ex(const gsp_csr *a, const float *x, int64_t f, int64_t ldx, float *y, int64_t ldy,
                                  const gsp_spmm_opts *opts, gsp_stream stream) {
  return spmm_impl(a, x, f, ldx, y, ldy, opts, GSP_REDUCE_SUM, cs(stream), "gsp_spmm_ex");
}

extern "C" gsp_status gsp_spmm_plan_info(const gsp_csr *a, const float *x, int64_t f, int64_t ldx,
                                         const gsp_spmm_opts *opts, int32_t *launches, int32_t *slab_cols,
                                         int32_t *tail_slab_cols) {
  clear_detail();
  gsp_status st = check_csr(a, false, "gsp_spmm_plan_info");
  if (st) return st;
  if (f < 0 || ldx < f) return fail(GSP_ERR_INVALID_ARG, "gsp_spmm_plan_info: need f >= 0, ldx >= f");
  SpmmPlan P{};
  if (a->n_rows == 0 || f == 0) {
    if (launches) *launches = 0;
    return GSP_OK;
  }
  if ((st = spmm_plan(a, x, f, ldx, opts, &P))) return st;
  if (launches) *launches = P.f_tail ? 2 : 1;
  if (slab_cols) *slab_cols = (int32_t)P.main.slab_cols;
  if (tail_slab_cols) *tail_slab_cols = P.f_tail ? (int32_t)P.tail.slab_cols : 0;
  return GSP_OK;
}

extern "C" gsp_status gsp_multihead_spmm(const gsp_csr *a, int32_t heads, const float *alpha, const float *z,
                                         int64_t d, int64_t ldz, float *y, int64_t ldy, gsp_stream stream) {
  const char *fn = "gsp_multihead_spmm";
  clear_detail();
  gsp_status st = check_csr(a, false, fn);
  if (st) return st;
  if (heads <= 0 || d < 0) return fail(GSP_ERR_INVALID_ARG, "%s: heads >= 1 and d >= 0 required", fn);
  const int64_t f = (int64_t)heads * d;
  if (ldz < f || ldy < f) return fail(GSP_ERR_INVALID_ARG, "%s: need ldz, ldy >= heads*d", fn);
  if (a->n_rows == 0 || f == 0) return GSP_OK;
  if (!y || (a->n_cols > 0 && !z) || (a->nnz > 0 && !alpha))
    return fail(GSP_ERR_INVALID_ARG, "%s: null pointer", fn);
  const size_t zb = a->n_cols ? (size_t)((a->n_cols - 1) * ldz + f) * 4 : 0;
  const size_t yb = (size_t)((a->n_rows - 1) * ldy + f) * 4;
  if (overlaps(z, zb, y, yb)) return fail(GSP_ERR_ALIAS, "%s: z and y overlap", fn);
  int vmax = 1;
  if (ldz % 4 == 0 && aligned16(z)) vmax = 4;
  else if (ldz % 2 == 0 && aligned8(z)) vmax = 2;
  EngineLaunch L;
  st = engine_plan(a->n_rows, a->n_cols, a->nnz, f, d, vmax, 0, 0, &L, kMaxHpt);
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
  if ((st = engine_ldxv(p, L, a->n_cols, ldz))) return st;
  return engine_launch(L, p, WeightAlpha{alpha, heads}, cs(stream));
}
