// spmm_engine.cuh -- the row-gather/reduce engine behind gsp_spmm,
// gsp_multihead_spmm and gsp_gat_aggregate (§4.1, Eq. formula:1,
// P:640-648; multi-head P:648-649; edge softmax P:653-656).
//
// Mapping (DESIGN.md §Kernels / K-spmm):
//  * Column SLABS.  The feature width is cut into slabs of SW = G*V columns.
//    The grid is slab-major (blockIdx = slab * nblk + blk) so at any moment
//    the resident CTAs gather from ONE slab of X, whose n x SW x 4 B footprint
//    is sized to stay resident in the 126 MB L2: every gathered row after the
//    first hit comes from L2 instead of HBM.
//  * nnz-balanced ROW BLOCKS (merge-path on row starts): CTA blk owns the rows
//    whose first nonzero lies in [blk*C, (blk+1)*C); its row range is found by
//    a warp-cooperative 33-ary search of row_ptr.
//  * A TEAM (a warp when G >= 8) owns one (row, slab).  It is split into
//    SPR = T/G sub-groups of G lanes; each lane holds V consecutive columns
//    (float4 when aligned), so one edge = one coalesced G*V*4-byte row-slab
//    read ("consecutive threads along the feature dimension"), and the
//    sub-groups take interleaved edges so a warp keeps 32 gathers in flight
//    without intra-warp divergence.
//  * Column indices and edge weights of a 32-edge SEGMENT are loaded once,
//    coalesced (lane l loads edge l), and broadcast by shuffle (the paper
//    caches them in shared memory; registers + SHFL are the sm_100a
//    equivalent without an smem round trip).
//  * Hub rows (degree > kHub) are processed by the whole CTA: the row is cut
//    into kVirt = 16 contiguous segment ranges whose partials are combined by
//    a fixed pairwise tree in shared memory.
//
// Summation order (depends only on the row, never on G, V, SW, C or the
// partition -> bitwise reproducible and partition-invariant):
//    segment = (r0 + r1) + (r2 + r3), r_k = fma chain over the segment's
//              edges j = k mod 4 (32-edge segments from the row start)
//    row sum = sequential sum of its segments           (degree <= kHub)
//    hub row = pairwise tree over 16 ranges; a range sums its segments into
//              acc1, folded into acc2 every 32 segments.
#pragma once

#include <cuda_fp16.h>

#include <type_traits>

#include "common.cuh"

namespace gsp {

constexpr int kThreads = 256;      // threads per CTA (8 warps)
constexpr int kSeg = 32;           // edges per segment
#ifndef GSP_UNROLL
#define GSP_UNROLL 8
#endif
constexpr int kUnroll = GSP_UNROLL;  // gathers in flight per lane
constexpr int kHub = 512;          // degree above which a row is CTA-cooperative
constexpr int kVirt = 16;          // virtual ranges of a hub row
constexpr int kMaxHubPerBlock = 64;
constexpr int kStageChunks = 4;   // TMA bulk-copy chunks of the CSR window
constexpr int kMaxHpt = 4;        // heads per team (multi-head modes)
#ifndef GSP_HM_U
#define GSP_HM_U 8
#endif
#ifndef GSP_MIN_BLOCKS
#define GSP_MIN_BLOCKS 4
#endif
constexpr int kMinBlocks = GSP_MIN_BLOCKS;  // CTAs per SM the register budget is sized for

// ----------------------------------------------------------------- vectors
template <int V>
struct Vec;
#ifndef GSP_L2HINT
#define GSP_L2HINT 0
#endif
// GSP_L2HINT=1: gathers of X carry an L2 evict_last policy and the staged CSR
// window evict_first, so the streamed CSR does not push X slabs out of L2.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
template <>
struct Vec<4> {
  static __device__ __forceinline__ void ld(float (&r)[4], const float *p) {
#if GSP_L2HINT
    float4 t;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(t.x), "=f"(t.y), "=f"(t.z), "=f"(t.w)
                 : "l"(p), "l"(l2_policy_evict_last()));
#else
    float4 t = __ldg(reinterpret_cast<const float4 *>(p));
#endif
    r[0] = t.x; r[1] = t.y; r[2] = t.z; r[3] = t.w;
  }
  static __device__ __forceinline__ void st(float *p, const float (&r)[4]) {
    __stcs(reinterpret_cast<float4 *>(p), make_float4(r[0], r[1], r[2], r[3]));
  }
  static __device__ __forceinline__ void st_shared(float *p, const float (&r)[4]) {
    *reinterpret_cast<float4 *>(p) = make_float4(r[0], r[1], r[2], r[3]);
  }
};
template <>
struct Vec<8> {  // two float4 per lane (256-column slabs)
  static __device__ __forceinline__ void ld(float (&r)[8], const float *p) {
    const float4 a = __ldg(reinterpret_cast<const float4 *>(p));
    const float4 b = __ldg(reinterpret_cast<const float4 *>(p) + 1);
    r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w;
    r[4] = b.x; r[5] = b.y; r[6] = b.z; r[7] = b.w;
  }
  static __device__ __forceinline__ void st(float *p, const float (&r)[8]) {
    __stcs(reinterpret_cast<float4 *>(p), make_float4(r[0], r[1], r[2], r[3]));
    __stcs(reinterpret_cast<float4 *>(p) + 1, make_float4(r[4], r[5], r[6], r[7]));
  }
};
template <>
struct Vec<2> {
  static __device__ __forceinline__ void ld(float (&r)[2], const float *p) {
    float2 t = __ldg(reinterpret_cast<const float2 *>(p));
    r[0] = t.x; r[1] = t.y;
  }
  static __device__ __forceinline__ void st(float *p, const float (&r)[2]) {
    __stcs(reinterpret_cast<float2 *>(p), make_float2(r[0], r[1]));
  }
  static __device__ __forceinline__ void st_shared(float *p, const float (&r)[2]) {
    *reinterpret_cast<float2 *>(p) = make_float2(r[0], r[1]);
  }
};
template <>
struct Vec<1> {
  static __device__ __forceinline__ void ld(float (&r)[1], const float *p) { r[0] = __ldg(p); }
  static __device__ __forceinline__ void st(float *p, const float (&r)[1]) { __stcs(p, r[0]); }
  static __device__ __forceinline__ void st_shared(float *p, const float (&r)[1]) { *p = r[0]; }
};

template <int V>
struct VecT;
template <>
struct VecT<8> { using T = float4; };  // addressed in float4 units (ldxv = ldx / 4)
template <>
struct VecT<4> { using T = float4; };
template <>
struct VecT<2> { using T = float2; };
template <>
struct VecT<1> { using T = float; };

template <int V>
__device__ __forceinline__ void vld(float (&r)[V], const typename VecT<V>::T *p) {
  Vec<V>::ld(r, reinterpret_cast<const float *>(p));
}

// ------------------------------------------------- feature element policies
// XE: how a lane's V features of one gathered row are stored in X.
//  XF32<V>: fp32 (float4 / float2 / float loads, the default);
//  XF16<V>: fp16 storage ("fp16" mixed precision): V = 8 halves
//           per 16-byte load (or 1), converted to fp32 at FMA time -- the
//           arithmetic stays fp32.
// Raw: what a gather lands in (registers); unpack() runs after all gathers of
// a chunk are issued, so conversion never stalls the loads.
template <int V>
struct XF32 {
  using Elem = float;
  using Ptr = typename VecT<V>::T;  // addressed in these units (ldxv = ldx / width)
  static constexpr int kWidth = V == 8 ? 4 : V;
  static constexpr int kU = V >= 8 ? (kUnroll < 4 ? kUnroll : 4) : kUnroll;  // gathers in flight per lane
  static constexpr int kMinBlocks = 0;                                        // engine default
  struct Raw {
    float v[V];
  };
  static __device__ __forceinline__ void ld(Raw &r, const Ptr *p) { vld<V>(r.v, p); }
  static __device__ __forceinline__ void zero(Raw &r) {
#pragma unroll
    for (int i = 0; i < V; ++i) r.v[i] = 0.0f;
  }
  static __device__ __forceinline__ void unpack(const Raw &r, float (&x)[V]) {
#pragma unroll
    for (int i = 0; i < V; ++i) x[i] = r.v[i];
  }
};
template <int V>
struct XF16;
#ifndef GSP_F16_MIN_BLOCKS
#define GSP_F16_MIN_BLOCKS 2
#endif
template <>
struct XF16<8> {
  using Elem = __half;
  using Ptr = uint4;
  static constexpr int kWidth = 8;
  static constexpr int kU = kUnroll;
  static constexpr int kMinBlocks = GSP_F16_MIN_BLOCKS;  // 8 fp32 accumulators x 4 residues per lane
  struct Raw {
    uint4 q;
  };
  static __device__ __forceinline__ void ld(Raw &r, const Ptr *p) { r.q = __ldg(p); }
  static __device__ __forceinline__ void zero(Raw &r) { r.q = make_uint4(0u, 0u, 0u, 0u); }
  static __device__ __forceinline__ void unpack(const Raw &r, float (&x)[8]) {
    const uint32_t w[4] = {r.q.x, r.q.y, r.q.z, r.q.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&w[i]));
      x[2 * i] = f.x;
      x[2 * i + 1] = f.y;
    }
  }
};
#ifndef GSP_F16_UNROLL
#define GSP_F16_UNROLL GSP_UNROLL
#endif
template <>
struct XF16<4> {
  using Elem = __half;
  using Ptr = uint2;
  static constexpr int kWidth = 4;
  static constexpr int kU = GSP_F16_UNROLL;
  static constexpr int kMinBlocks = 0;
  struct Raw {
    uint2 q;
  };
  static __device__ __forceinline__ void ld(Raw &r, const Ptr *p) { r.q = __ldg(p); }
  static __device__ __forceinline__ void zero(Raw &r) { r.q = make_uint2(0u, 0u); }
  static __device__ __forceinline__ void unpack(const Raw &r, float (&x)[4]) {
    const uint32_t w[2] = {r.q.x, r.q.y};
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&w[i]));
      x[2 * i] = f.x;
      x[2 * i + 1] = f.y;
    }
  }
};
template <>
struct XF16<1> {
  using Elem = __half;
  using Ptr = __half;
  static constexpr int kWidth = 1;
  static constexpr int kU = kUnroll;
  static constexpr int kMinBlocks = 0;
  struct Raw {
    __half h;
  };
  static __device__ __forceinline__ void ld(Raw &r, const Ptr *p) { r.h = __ldg(p); }
  static __device__ __forceinline__ void zero(Raw &r) { r.h = __float2half(0.0f); }
  static __device__ __forceinline__ void unpack(const Raw &r, float (&x)[1]) { x[0] = __half2float(r.h); }
};

// Store V values of which the first nvalid are real columns.
template <int V>
__device__ __forceinline__ void store_cols(float *p, const float (&r)[V], int nvalid, bool vec_ok) {
  if (nvalid >= V && vec_ok) {
    Vec<V>::st(p, r);
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i)
      if (i < nvalid) __stcs(p + i, r[i]);
  }
}

// ------------------------------------------------------- staged CSR window
// Entries [wb, we) of col (and val when staged) live in shared memory, copied
// by the TMA engine at CTA start (cp.async.bulk, 4 chunks, one mbarrier each);
// anything outside the window (hub rows reaching past it, misaligned arrays)
// is read from global memory with streaming loads.
struct Window {
  const int32_t *scol;
  const float *sval;  // NULL when values are not staged
  const float *swt;   // per-head weights [hpt][cap] staged by TMA (WeightAlphaHM), else NULL
  int64_t cap;        // window capacity (entries)
  int64_t wb, we;
  __device__ __forceinline__ bool in(int64_t e) const { return e >= wb && e < we; }
  __device__ __forceinline__ int col(const int32_t *g, int64_t e) const { return in(e) ? scol[e - wb] : __ldcs(g + e); }
  __device__ __forceinline__ float val(const float *g, int64_t e) const {
    return (sval && in(e)) ? sval[e - wb] : __ldcs(g + e);
  }
};

// ---------------------------------------------------------- reduce policies
// phi of Eq. formula:1: sum (also mean = sum / row count) or the
// row-wise max / min of psi(x, w) = w * x ("min and max as reduce").
struct RedSum {
  static constexpr bool kSum = true;
  static __device__ __forceinline__ float init() { return 0.0f; }
  static __device__ __forceinline__ float step(float acc, float w, float x) { return fmaf(w, x, acc); }
  static __device__ __forceinline__ float comb(float a, float b) { return a + b; }
};
struct RedMax {
  static constexpr bool kSum = false;
  static __device__ __forceinline__ float init() { return -INFINITY; }
  static __device__ __forceinline__ float step(float acc, float w, float x) { return fmaxf(acc, w * x); }
  static __device__ __forceinline__ float comb(float a, float b) { return fmaxf(a, b); }
};
struct RedMin {
  static constexpr bool kSum = false;
  static __device__ __forceinline__ float init() { return INFINITY; }
  static __device__ __forceinline__ float step(float acc, float w, float x) { return fminf(acc, w * x); }
  static __device__ __forceinline__ float comb(float a, float b) { return fminf(a, b); }
};

// ---------------------------------------------------------- weight functors
// Each functor provides Row row(int64 r, int head) and Row::w(e, c): the
// weight of CSR entry e (column c) for this group's head.

// kUnit: every weight is 1 (no weight array); kComputed: the weight needs
// arithmetic (made once per edge by the team into shared scratch); otherwise
// the weight is a stored value (staged with the window when possible).
struct WeightVal {  // SpMM with A's values
  const float *val;
  struct Row {
    static constexpr bool kUnit = false, kComputed = false, kStagedVal = true, kMultiHead = false, kInStats = false;
    const float *val;
    __device__ __forceinline__ float w(int64_t e, int /*c*/, int /*hh*/) const { return __ldcs(val + e); }
  };
  __device__ __forceinline__ Row row(int64_t, int, bool, void *) const { return Row{val}; }
};

struct WeightOne {  // SpMM with val == NULL: psi = copy
  struct Row {
    static constexpr bool kUnit = true, kComputed = false, kStagedVal = false, kMultiHead = false, kInStats = false;
    __device__ __forceinline__ float w(int64_t, int, int) const { return 1.0f; }
  };
  __device__ __forceinline__ Row row(int64_t, int, bool, void *) const { return Row{}; }
};

struct WeightAlpha {  // multi-head SpMM with given alpha [nnz][H]
  const float *alpha;
  int heads;
  struct Row {
    static constexpr bool kUnit = false, kComputed = false, kStagedVal = false, kMultiHead = true, kInStats = false;
    const float *alpha;
    int heads, h;  // h: first head of the team's slab
    __device__ __forceinline__ float w(int64_t e, int, int hh) const { return __ldcs(alpha + e * heads + h + hh); }
  };
  __device__ __forceinline__ Row row(int64_t, int h, bool, void *) const { return Row{alpha, heads, h}; }
};

// Multi-head SpMM with alpha HEAD-MAJOR [H][ahs] (the fused GAT's two-launch
// schedule writes it so; ahs = nnz rounded up to 32): the window's weights of
// the slab's hpt heads are staged by the TMA engine with the column indices
// (one contiguous run per head), so the gather loop reads weights from shared
// memory with no per-segment loads; hub rows beyond the window read them from
// global memory.
struct WeightAlphaHM {
  const float *alpha;
  int64_t ahs;
  struct Row {
    static constexpr bool kUnit = false, kComputed = false, kStagedVal = false, kMultiHead = true, kInStats = false;
    static constexpr bool kStagedHeads = true;
    const float *alpha;
    int64_t ahs;
    int h;  // first head of the team's slab
    __device__ __forceinline__ float w(int64_t e, int, int hh) const { return __ldcs(alpha + (h + hh) * ahs + e); }
  };
  __device__ __forceinline__ Row row(int64_t, int h, bool, void *) const { return Row{alpha, ahs, h}; }
};

template <class R, class = void>
struct HasStagedHeads : std::false_type {};
template <class R>
struct HasStagedHeads<R, std::void_t<decltype(R::kStagedHeads)>> : std::bool_constant<R::kStagedHeads> {};

struct GatStat {  // per (row, head) softmax statistics (standalone edge softmax)
  double m;       // row max of the score (fp64)
  float inv_s;    // 1 / sum exp(s - m)
  float pad;
};

// Fused GAT weight (A13): s = LeakyReLU(el[u] + er[v]) in fp64,
// alpha = exp(s - m) / S with the row statistics (m, S) of the (row, head).
//  kPre = false: the statistics are reduced inside the aggregate kernel by
//    the team that owns the (row, head) (single launch; one head per team, the
//    fp64 row state in registers).
//  kPre = true : the statistics come precomputed from row_stats_warp (gat.cu;
//    one warp per row for all heads) through st[n_rows][H]; the aggregate
//    kernel only forms alpha on the fly (never materialised).
template <bool kPre>
struct WeightGatT {
  const float *el, *er;
  float *alpha_out;
  double slope;
  int heads;
  const GatStat *st;  // kPre only
  struct Row {
    // kPre: a team may own several whole heads (slab = hpt heads); the Row of
    // a lane is that of the lane's own head, and the lanes of a head make
    // that head's weights (see row_segments)
    static constexpr bool kUnit = false, kComputed = true, kStagedVal = false, kMultiHead = kPre, kInStats = !kPre;
    const float *er;
    float *alpha_out;
    double el_u, m, slope;
    float inv_s;
    int heads, h;
    __device__ __forceinline__ double score(int c, int = 0) const {
      const double t = el_u + (double)__ldg(er + (int64_t)c * heads + h);
      return t >= 0.0 ? t : slope * t;
    }
    __device__ __forceinline__ float finish(int64_t e, double s, int = 0) const {
      const float a = expf((float)(s - m)) * inv_s;
      if (alpha_out) alpha_out[e * heads + h] = a;
      return a;
    }
  };
  // h: the head of the calling lane; first_slab: only the first slab of a
  // head writes alpha_out (each entry once)
  __device__ __forceinline__ Row row(int64_t r, int h, bool first_slab, void *) const {
    Row w{er, first_slab ? alpha_out : nullptr, (double)__ldg(el + r * heads + h), 0.0, slope, 0.0f, heads, h};
    if constexpr (kPre) {
      const GatStat *g = st + r * heads + h;
      w.m = __ldg(&g->m);
      w.inv_s = __ldg(&g->inv_s);
    }
    return w;
  }
};
using WeightGat = WeightGatT<false>;
using WeightGatPre = WeightGatT<true>;

// ------------------------------------------------------------------ params
struct EngineParams {
  const int64_t *row_ptr;
  const int32_t *col;
  const void *x;  // fp32 (XF32) or fp16 (XF16) features
  float *y;
  int64_t n_rows, ldx, ldy, f;
  uint32_t ldxv;  // ldx / V: row stride of x in V-wide vectors (32-bit gather offsets)
  int64_t block_nnz, nblk;
  int64_t head_dim;  // D for multi-head modes (slabs never straddle heads); 0 = no heads
  int y_vec_ok;      // y base and ldy allow V-wide stores
  int64_t nnz;
  const float *stage_val;  // val array to stage in smem (NULL: none)
  const float *stage_hm;   // head-major weights to stage per slab head (WeightAlphaHM), NULL: none
  int64_t stage_hm_stride; // elements between heads of stage_hm
  int stage_heads;         // heads staged per slab (= hpt) when stage_hm
  int stage;               // 1: stage col (and stage_val) in shared memory
  int win_cap;             // window capacity in entries (multiple of 4)
  int mean;                // GSpMM mean: divide the row sum by the row's entry count
  int hpt;                 // heads per team (slab = hpt whole heads); 1 otherwise
  // fused accumulate epilogue (K-step propagation): acc = acc_coef * out +
  // (acc_src ? src_coef * acc_src : acc); y is not written when skip_y
  float *acc;
  const float *acc_src;
  int64_t ldacc, ldsrc;
  float acc_coef, src_coef;
  int skip_y, acc_vec_ok, src_vec_ok;
  // fused layer epilogue (NEXT-1): out = act(out + bias[col]); act 0 none, 1 ReLU, 2 ELU
  const float *bias;
  int act;
};

template <int V>
__device__ __forceinline__ void load_cols(float (&r)[V], const float *p, int nvalid, bool vec_ok) {
  if (nvalid >= V && vec_ok) {
    Vec<V>::ld(r, p);
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) r[i] = i < nvalid ? p[i] : 0.0f;
  }
}

// Row epilogue: store out[] to y and/or fold it into the accumulator.
template <int V>
__device__ __forceinline__ void epilogue(const EngineParams &p, int64_t r, int64_t col0, const float (&out_in)[V],
                                         int nvalid) {
  if (!p.bias && p.act == 0 && !p.acc) {  // plain Y = A X (uniform branch)
    if (!p.skip_y) store_cols<V>(p.y + r * p.ldy + col0, out_in, nvalid, p.y_vec_ok);
    return;
  }
  float out[V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    float v = out_in[i];
    if (p.bias && i < nvalid) v += __ldg(p.bias + col0 + i);
    if (p.act == 1) v = fmaxf(v, 0.0f);
    else if (p.act == 2) v = v > 0.0f ? v : expm1f(v);
    out[i] = v;
  }
  if (p.acc) {
    float prev[V], nv[V];
    if (p.acc_src) {
      load_cols<V>(prev, p.acc_src + r * p.ldsrc + col0, nvalid, p.src_vec_ok);
#pragma unroll
      for (int i = 0; i < V; ++i) prev[i] *= p.src_coef;
    } else {
      load_cols<V>(prev, p.acc + r * p.ldacc + col0, nvalid, p.acc_vec_ok);
    }
#pragma unroll
    for (int i = 0; i < V; ++i) nv[i] = fmaf(p.acc_coef, out[i], prev[i]);
    store_cols<V>(p.acc + r * p.ldacc + col0, nv, nvalid, p.acc_vec_ok);
  }
  if (!p.skip_y) store_cols<V>(p.y + r * p.ldy + col0, out, nvalid, p.y_vec_ok);
}

// Team geometry.  A TEAM of T lanes owns one (row, slab): T = 32 when the
// group width G >= 8 (a whole warp per row), else 4G (several rows per warp).
// The team holds SPR = T/G sub-groups; each sub-group covers the slab's SW
// columns and processes every SPR-th edge of a segment.
template <int G>
struct Team {
  static constexpr int T = (G >= 8) ? 32 : 4 * G;
  static constexpr int SPR = T / G;        // sub-groups per team: 1, 2 or 4
  static constexpr int NACC = 4 / SPR;     // residue accumulators per sub-group
  static constexpr int EPL = kSeg / T;     // metadata entries per lane per segment
  static constexpr int EPS = kSeg / SPR;   // edges per sub-group per segment
  static constexpr int U = EPS < kUnroll ? EPS : kUnroll;
};

template <int T>
__device__ __forceinline__ double team_max(double v, unsigned tmask) {
#pragma unroll
  for (int o = 1; o < T; o <<= 1) v = fmax(v, __shfl_xor_sync(tmask, v, o, T));
  return v;
}
template <int T>
__device__ __forceinline__ double team_sum(double v, unsigned tmask) {  // xor butterfly: fixed order, all lanes equal
#pragma unroll
  for (int o = 1; o < T; o <<= 1) v += __shfl_xor_sync(tmask, v, o, T);
  return v;
}

// Gather + FMA over one segment whose metadata is in shared memory (sc: 32
// column indices, sw: 32 weights, unused when Row::kUnit).  kFull: cnt == 32.
template <int V, int G, class Row, class R, bool kFull, class XE, class Pre>
__device__ __forceinline__ void seg_gather(const int32_t *sc, const float *sw, int cnt,
                                           const typename XE::Ptr *__restrict__ xb, uint32_t ldxv, int nact,
                                           int sg, float (&a)[Team<G>::NACC][V], Pre &&pre) {
  using TM = Team<G>;
  constexpr int SPR = TM::SPR, NACC = TM::NACC, EPS = TM::EPS;
  // gathers in flight per lane: the element policy's budget; the single-launch
  // GAT (in-kernel statistics, fp64 row state live) measured best at 4
  constexpr int kUx = Row::kInStats ? (XE::kU < 4 ? XE::kU : 4)
                      : HasStagedHeads<Row>::value ? (XE::kU < GSP_HM_U ? XE::kU : GSP_HM_U)
                                                   : XE::kU;
  constexpr int U = TM::U < kUx ? TM::U : kUx;
  using Raw = typename XE::Raw;
  static_assert(EPS % U == 0, "GSP_UNROLL must divide the edges per sub-group and segment (power of two)");
  (void)nact;
  auto load = [&](int t0, Raw (&xv)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = sg + SPR * (t0 + u);
      const bool ok = kFull || j < cnt;
      const uint32_t cj = ok ? (uint32_t)sc[j] : 0u;
      // the last vector of a row-slab may cover ld padding (x is [n_cols][ldx],
      // gsp.h): those columns are read whole and their sums never stored.
      // Lanes past f (nact == 0) read the last valid vector (xb is clamped
      // there): same sectors as an active lane, no predicate, never stored.
      if (ok) {
        XE::ld(xv[u], xb + cj * ldxv);
      } else {
        XE::zero(xv[u]);
      }
    }
  };
  auto fma = [&](int t0, const Raw (&xv)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t0 + u;
      const int j = sg + SPR * t;
      if (kFull || j < cnt) {
        const float ww = Row::kUnit ? 1.0f : sw[j];
        float xf[V];
        XE::unpack(xv[u], xf);
#pragma unroll
        for (int i = 0; i < V; ++i) a[t % NACC][i] = R::step(a[t % NACC][i], ww, xf[i]);
      }
    }
  };
  {
#pragma unroll
    for (int t0 = 0; t0 < EPS; t0 += U) {
      if (!kFull && SPR * t0 >= cnt) break;
      Raw xv[U];
      load(t0, xv);
      // the first chunk's gathers are in flight: now make the weights (team-
      // uniform hook; fills sw when the weights need arithmetic or loads)
      if (t0 == 0) pre();
      fma(t0, xv);
    }
  }
}

// Accumulate segments [s_begin, s_end) of the row starting at `start` (degree
// d) into out[V].  Canonical order (independent of G, V, T):
//   residue chain r_k = fma chain, from 0, over the segment's edges j with
//                       j % 4 == k, in increasing j
//   segment sum       = (r_0 + r_1) + (r_2 + r_3)
//   acc1 += segment (sequential); every 32 segments acc2 += acc1, acc1 = 0
//   out = acc2 + acc1 (kLong: hub ranges) or acc1 (rows of <= kHub edges,
//   i.e. <= 16 segments, where acc2 would stay 0)
// Every lane of the team ends with the same out[] (all sub-groups combine).
// Metadata: segments inside the TMA-staged window are read from it directly;
// other segments (hub rows beyond the window, unstaged arrays) and computed
// weights go through the team's 32-entry shared scratch (tc, tw).
template <int V, int G, bool kLong, class R, class XE, class Row, class Pro>
__device__ __forceinline__ void row_segments(const EngineParams &p, const Window &win, Row &wr, int64_t start,
                                             int64_t d, int64_t s_begin, int64_t s_end,
                                             const typename XE::Ptr *__restrict__ xb, int nact, int tl, int sg,
                                             unsigned tmask, int32_t *tc, float *tw, int hl, const double *cache,
                                             int ncache, float (&out)[V], Pro &&prologue) {
  using TM = Team<G>;
  constexpr int T = TM::T, SPR = TM::SPR, NACC = TM::NACC, EPL = TM::EPL;
  float acc1[V], acc2[V];
#pragma unroll
  for (int i = 0; i < V; ++i) acc1[i] = acc2[i] = R::init();
  int n1 = 0;
  for (int64_t s = s_begin; s < s_end; ++s) {
    const int64_t e0 = start + s * kSeg;
    const int cnt = (int)(d - s * kSeg < kSeg ? d - s * kSeg : kSeg);
    const bool seg_in = win.in(e0) && e0 + cnt <= win.we;  // team-uniform
    const int32_t *sc;
    const float *sw = tw + hl * kSeg;  // this lane's head's weights
    bool scratch = false;
    if (seg_in) {
      sc = win.scol + (e0 - win.wb);
      if (Row::kStagedVal && win.sval) sw = win.sval + (e0 - win.wb);
      else if (HasStagedHeads<Row>::value && win.swt) sw = win.swt + hl * win.cap + (e0 - win.wb);
      else scratch = !Row::kUnit;
    } else {
      sc = tc;
      scratch = true;
    }
    if (!seg_in) {  // column indices from global memory into the team scratch
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const int j = tl + T * i;
        if (j < cnt) tc[j] = __ldcs(p.col + e0 + j);
      }
      __syncwarp(tmask);
    }
    // weights are made while the first chunk of gathers is in flight
    const bool first = (s == s_begin);
    auto pre = [&]() {
      if (first) prologue();
      if constexpr (Row::kComputed && Row::kMultiHead) {
        // the T/hpt lanes of head hl make that head's weights: lane of rank k
        // among them makes entries k, k + T/hpt, ... (its Row is its head's)
        const int gph = G / p.hpt;                      // lanes of a head per sub-group
        const int rank = sg * gph + (tl % G) % gph;     // rank among the head's lanes
        for (int j = rank; j < cnt; j += T / p.hpt) tw[hl * kSeg + j] = wr.finish(e0 + j, wr.score(sc[j]));
        __syncwarp(tmask);
      } else if (scratch && !Row::kUnit) {  // cooperative: lane tl makes entries tl + T*i
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          const int j = tl + T * i;
          if (j < cnt) {
            const int c = sc[j];
            const int64_t q = e0 + j - start;  // row-relative; cached by this same lane
            constexpr int kHH = Row::kMultiHead ? kMaxHpt : 1;  // single-head modes: compile-time 1
#pragma unroll
            for (int hh = 0; hh < kHH; ++hh) {
              if (hh == 0 || hh < p.hpt) {
                if constexpr (Row::kComputed)
                  tw[j] = wr.finish(e0 + j, (cache && q < ncache) ? cache[q] : wr.score(c));
                else
                  tw[hh * kSeg + j] = wr.w(e0 + j, c, hh);
              }
            }
          }
        }
        __syncwarp(tmask);
      }
    };
    float a[NACC][V];
#pragma unroll
    for (int q = 0; q < NACC; ++q)
#pragma unroll
      for (int i = 0; i < V; ++i) a[q][i] = R::init();
    if (cnt == kSeg) seg_gather<V, G, Row, R, true, XE>(sc, sw, cnt, xb, p.ldxv, nact, sg, a, pre);
    else seg_gather<V, G, Row, R, false, XE>(sc, sw, cnt, xb, p.ldxv, nact, sg, a, pre);
    if (scratch) __syncwarp(tmask);  // scratch is rewritten by the next segment
    // segment sum (r0 + r1) + (r2 + r3); residue k lives in sub-group k % SPR,
    // accumulator k / SPR
    float seg[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
      if (SPR == 1) {
        seg[i] = R::comb(R::comb(a[0][i], a[1 % NACC][i]), R::comb(a[2 % NACC][i], a[3 % NACC][i]));
      } else if (SPR == 2) {
        const float b0 = R::comb(a[0][i], __shfl_xor_sync(tmask, a[0][i], G, T));
        const float b1 = R::comb(a[NACC - 1][i], __shfl_xor_sync(tmask, a[NACC - 1][i], G, T));
        seg[i] = R::comb(b0, b1);
      } else {
        const float b = R::comb(a[0][i], __shfl_xor_sync(tmask, a[0][i], G, T));
        seg[i] = R::comb(b, __shfl_xor_sync(tmask, b, 2 * G, T));
      }
    }
#pragma unroll
    for (int i = 0; i < V; ++i) acc1[i] = R::comb(acc1[i], seg[i]);
    if (kLong && ++n1 == kSeg) {
#pragma unroll
      for (int i = 0; i < V; ++i) {
        acc2[i] = R::comb(acc2[i], acc1[i]);
        acc1[i] = R::init();
      }
      n1 = 0;
    }
  }
#pragma unroll
  for (int i = 0; i < V; ++i) out[i] = kLong ? R::comb(acc2[i], acc1[i]) : acc1[i];
}

// epilogue: empty rows give 0 for every reduce; mean divides by the
// row's entry count
template <class R, int V>
__device__ __forceinline__ void finish_row(float (&out)[V], int64_t d, int mean) {
#pragma unroll
  for (int i = 0; i < V; ++i) {
    if (d == 0) out[i] = 0.0f;
    else if (R::kSum && mean) out[i] = out[i] / (float)d;
  }
}

// register budget: 4 CTAs/SM (64 regs) for stored/unit weights and the
// single-launch GAT weight; 3 CTAs/SM (85 regs) for multi-head computed GAT
// weights (precomputed statistics)
#ifndef GSP_GAT_MIN_BLOCKS
#define GSP_GAT_MIN_BLOCKS 4
#endif
#ifndef GSP_GATPRE_MIN_BLOCKS
#define GSP_GATPRE_MIN_BLOCKS 3
#endif
// multi-head SpMM with stored alpha (WeightAlpha) and the fused GAT's staged
// head-major alpha (WeightAlphaHM): 3 CTAs/SM (85 registers).  At 64 registers
// the per-lane head offset and weight pointers spill inside the segment loop
// (120 / 152 B of local stores / loads); measured on C3 (8 x 64): fused GAT
// 0.532 -> 0.452 ms, multi-head SpMM 0.456 -> 0.427 ms (C2g 8 x 64: +-5%,
// tools/c3_probe.py)
#ifndef GSP_HM_MIN_BLOCKS
#define GSP_HM_MIN_BLOCKS 3
#endif
#ifndef GSP_MH_MIN_BLOCKS
#define GSP_MH_MIN_BLOCKS 3
#endif
template <class W, class XE>
struct MinBlocksFor {  // measured on C3 (8 x 64): multi-head computed weights 0.74 -> 0.67 ms at 3 CTAs/SM
  static constexpr int value = XE::kMinBlocks ? XE::kMinBlocks
                               : HasStagedHeads<typename W::Row>::value ? GSP_HM_MIN_BLOCKS
                               : (W::Row::kMultiHead && !W::Row::kComputed) ? GSP_MH_MIN_BLOCKS
                               : !W::Row::kComputed ? kMinBlocks
                               : (W::Row::kMultiHead ? GSP_GATPRE_MIN_BLOCKS : GSP_GAT_MIN_BLOCKS);
};

template <int V, int G, class W, class R, class XE = XF32<V>>
__global__ void __launch_bounds__(kThreads, MinBlocksFor<W, XE>::value) engine_kernel(const EngineParams p, const W wf) {
  using TM = Team<G>;
  constexpr int T = TM::T;
  constexpr int NT = kThreads / T;  // teams per CTA
  constexpr int SW = G * V;         // slab width (columns)
  __shared__ int64_t s_rb[2];
  __shared__ int s_hub[kMaxHubPerBlock];
  __shared__ int s_nhub, s_next;
  __shared__ __align__(16) float s_part[kVirt * SW];
  __shared__ __align__(8) uint64_t s_bar[kStageChunks];
  constexpr bool kMH = W::Row::kMultiHead;
  constexpr int kHptCap = (kMH && G >= 2) ? kMaxHpt : 1;  // G == 1 slabs never hold more than one head
  __shared__ float s_tw[NT][kHptCap * kSeg];              // per-team scratch: weights, per head
  __shared__ int32_t s_tc[NT][kSeg];  // per-team scratch: column indices
  using RowT = decltype(wf.row(0, 0, false, nullptr));
  constexpr bool kGat = RowT::kInStats;                         // in-kernel softmax statistics
  constexpr bool kMHC = RowT::kMultiHead && RowT::kComputed;    // per-lane head Rows (multi-head computed weights)
  constexpr int kCache = kGat ? 1024 / NT : 1;  // per-team fp64 score cache (GAT)
  __shared__ double s_cache[NT][kCache];
  __shared__ double s_red[kThreads / 32];
  __shared__ int64_t s_win[3];  // wb, we, chunk
  extern __shared__ __align__(16) uint8_t s_dyn[];  // staged col [win_cap] then val [win_cap]

  const int64_t blk = blockIdx.x % p.nblk;
  const int64_t slab = blockIdx.x / p.nblk;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int team = tid / T, tl = tid % T;
  const int sg = tl / G, gl = tl % G;
  const unsigned tmask = (T == 32) ? 0xffffffffu : (((1u << T) - 1u) << ((lane / T) * T));

  if (warp < 2) {
    const int64_t t = (blk + warp) * p.block_nnz;
    const int64_t r = warp_lower_bound(p.row_ptr, p.n_rows, t);
    if (lane == 0) s_rb[warp] = r;
  }
  if (tid == 0) {
    s_nhub = 0;
    s_next = 0;
    if (p.stage) {
#pragma unroll
      for (int k = 0; k < kStageChunks; ++k) mbar_init(&s_bar[k], 1);
      fence_mbar_init();
    }
  }
  __syncthreads();
  const int64_t rbeg = s_rb[0];
  const int64_t rend = (blk == p.nblk - 1) ? p.n_rows : s_rb[1];
  int32_t *s_col = reinterpret_cast<int32_t *>(s_dyn);
  float *s_val = reinterpret_cast<float *>(s_dyn + (size_t)p.win_cap * 4);
  // staged per-head weights (WeightAlphaHM): [stage_heads][win_cap] after col (and val)
  float *s_wt = reinterpret_cast<float *>(s_dyn + (size_t)p.win_cap * 4 * (p.stage_val ? 2 : 1));
  const int head = p.head_dim ? (int)((slab * SW) / p.head_dim) : 0;  // first head of the slab
  const int nst = (p.stage && p.stage_hm) ? p.stage_heads : 0;         // weight arrays staged per chunk

  // 0. TMA: stage the CSR window [wb, we) -- every non-hub row of this block
  //    lies inside [row_ptr[rbeg], row_ptr[rbeg] + block_nnz + kHub)
  if (tid == 0) {
    int64_t wb = 0, we = 0, ch = 1;
    if (p.stage && rbeg < rend) {
      const int64_t s0 = __ldg(p.row_ptr + rbeg);
      wb = s0 & ~int64_t(3);
      we = min(min(p.nnz, s0 + p.block_nnz + kHub), wb + (int64_t)p.win_cap) & ~int64_t(3);
      if (we < wb) we = wb;
      ch = (((we - wb + kStageChunks - 1) / kStageChunks) + 3) & ~int64_t(3);
      if (ch == 0) ch = 4;
      for (int k = 0; k < kStageChunks; ++k) {
        const int64_t c0 = wb + k * ch, c1 = min(we, c0 + ch);
        const uint32_t n = c1 > c0 ? (uint32_t)(c1 - c0) : 0u;
        const uint32_t bytes = n * 4u * ((p.stage_val ? 2u : 1u) + (uint32_t)nst);
        mbar_arrive_expect_tx(&s_bar[k], bytes);
        if (n) {
          bulk_g2s(s_col + (c0 - wb), p.col + c0, n * 4u, &s_bar[k]);
          if (p.stage_val) bulk_g2s(s_val + (c0 - wb), p.stage_val + c0, n * 4u, &s_bar[k]);
          for (int hh = 0; hh < nst; ++hh)
            bulk_g2s(s_wt + (size_t)hh * p.win_cap + (c0 - wb), p.stage_hm + (int64_t)(head + hh) * p.stage_hm_stride + c0,
                     n * 4u, &s_bar[k]);
        }
      }
    }
    s_win[0] = wb;
    s_win[1] = we;
    s_win[2] = ch;
  }

  // columns of this lane (identical for every sub-group of a team)
  const int64_t col0 = slab * SW + (int64_t)gl * V;
  const bool active = col0 < p.f;
  const int nvalid = (int)(p.f - col0 < V ? p.f - col0 : V);
  const int nact = active ? nvalid : 0;  // columns this lane gathers
  const int64_t last_vec = p.f > 0 ? ((p.f - 1) / V) * V : 0;  // first column of the last valid vector
  const auto *xb = reinterpret_cast<const typename XE::Ptr *>(reinterpret_cast<const typename XE::Elem *>(p.x) +
                                                                (active ? col0 : last_vec));
  const int hl = (kMH && p.hpt > 1) ? (int)((gl * V) / p.head_dim) : 0;  // this lane's head offset
  const bool first_slab = p.head_dim ? ((slab * SW) % p.head_dim) == 0 : true;

  // 1. collect hub rows
  for (int64_t r = rbeg + tid; r < rend; r += kThreads) {
    const int64_t d = __ldg(p.row_ptr + r + 1) - __ldg(p.row_ptr + r);
    if (d > kHub) {
      const int k = atomicAdd(&s_nhub, 1);
      if (k < kMaxHubPerBlock) s_hub[k] = (int)(r - rbeg);
    }
  }
  __syncthreads();
  const int nhub = s_nhub;  // <= kMaxHubPerBlock by the host's block_nnz cap
  const Window win{s_col, p.stage_val ? s_val : nullptr, nst ? s_wt : nullptr, p.win_cap, s_win[0], s_win[1]};
  const int64_t wchunk = s_win[2];
  int ready = 0;  // chunks this thread has seen complete
#ifndef GSP_WINDOW_PER_ROW_WAIT
  // every thread waits for the whole window, then a CTA barrier: measured as
  // fast as per-row chunk waits (C3 / C4 / C5 within noise) and it orders the
  // TMA writes before every read for compute-sanitizer's racecheck too
  if (p.stage)
    for (; ready < kStageChunks && win.wb + ready * wchunk < win.we; ++ready) mbar_wait(&s_bar[ready], 0);
  __syncthreads();
#endif
  // wait until the window covers [.., e_end) (or all of it)
  auto ensure = [&](int64_t e_end) {
    if (!p.stage) return;
    while (ready < kStageChunks && win.wb + ready * wchunk < min(e_end, win.we)) {
      mbar_wait(&s_bar[ready], 0);
      ++ready;
    }
  };

  // 2. hub rows: all teams cooperate; 16 virtual ranges, pairwise tree
  for (int k = 0; k < nhub; ++k) {
    const int64_t r = rbeg + s_hub[k];
    const int64_t start = __ldg(p.row_ptr + r);
    const int64_t d = __ldg(p.row_ptr + r + 1) - start;
    const int64_t S = (d + kSeg - 1) / kSeg;
    auto wr = wf.row(r, kMHC ? head + hl : head, first_slab, nullptr);
    ensure(start + d);
    if constexpr (kGat) {
      // CTA-wide softmax statistics of a hub row: thread tid takes edges
      // tid + 256k; warp xor butterflies, then warps 0..7 in order (fixed)
      double m = -INFINITY;
      for (int64_t q = tid; q < d; q += kThreads) m = fmax(m, wr.score(win.col(p.col, start + q)));
      m = team_max<32>(m, 0xffffffffu);
      if (lane == 0) s_red[warp] = m;
      __syncthreads();
      m = s_red[0];
      for (int w2 = 1; w2 < kThreads / 32; ++w2) m = fmax(m, s_red[w2]);
      __syncthreads();
      double S = 0.0;
      for (int64_t q = tid; q < d; q += kThreads)
        S += (double)expf((float)(wr.score(win.col(p.col, start + q)) - m));
      S = team_sum<32>(S, 0xffffffffu);
      if (lane == 0) s_red[warp] = S;
      __syncthreads();
      S = s_red[0];
      for (int w2 = 1; w2 < kThreads / 32; ++w2) S += s_red[w2];
      __syncthreads();
      wr.m = m;
      wr.inv_s = (float)(1.0 / S);
    }
    for (int v = team; v < kVirt; v += NT) {
      float part[V];
      row_segments<V, G, true, R, XE>(p, win, wr, start, d, (S * v) / kVirt, (S * (v + 1)) / kVirt, xb, nact, tl, sg, tmask,
                                  s_tc[team], s_tw[team], hl, nullptr, 0, part, [] {});
      if (sg == 0) {
#pragma unroll
        for (int i = 0; i < V; ++i) s_part[v * SW + gl * V + i] = part[i];
      }
    }
    __syncthreads();
#pragma unroll
    for (int stride = 1; stride < kVirt; stride <<= 1) {
      for (int q = tid; q < (kVirt / (2 * stride)) * SW; q += kThreads) {
        const int v = (q / SW) * 2 * stride, cidx = q % SW;
        s_part[v * SW + cidx] = R::comb(s_part[v * SW + cidx], s_part[(v + stride) * SW + cidx]);
      }
      __syncthreads();
    }
    if (team == 0 && sg == 0 && active) {
      float out[V];
#pragma unroll
      for (int i = 0; i < V; ++i) out[i] = s_part[gl * V + i];
      finish_row<R, V>(out, d, p.mean);
      epilogue<V>(p, r, col0, out, nvalid);
    }
    __syncthreads();
  }

  // 3. remaining rows: dynamic assignment, one team per row
  for (;;) {
    int k = 0;
    if (tl == 0) k = atomicAdd(&s_next, 1);
    k = __shfl_sync(tmask, k, 0, T);
    const int64_t r = rbeg + k;
    if (r >= rend) break;
    const int64_t start = __ldg(p.row_ptr + r);
    const int64_t d = __ldg(p.row_ptr + r + 1) - start;
    if (d > kHub) continue;
    auto wr = wf.row(r, kMHC ? head + hl : head, first_slab, nullptr);
    ensure(start + d);
    // GAT: the team's softmax statistics run inside the first segment, after
    // its first chunk of Z gathers has been issued; scores of the first kCache
    // edges are cached in fp64 by the lane that later turns them into alpha
    auto stats = [&]() {
      if constexpr (kGat) {
        // lane tl owns edges tl + T*k; the scores of the first kCache edges are
        // cached in fp64 by the lane that later turns them into alpha
        double m = -INFINITY;
        for (int64_t q = tl; q < d; q += T) {
          const double sc = wr.score(win.col(p.col, start + q));
          if (q < kCache) s_cache[team][q] = sc;
          m = fmax(m, sc);
        }
        m = team_max<T>(m, tmask);
        double S = 0.0;
        for (int64_t q = tl; q < d; q += T) {
          const double sc = q < kCache ? s_cache[team][q] : wr.score(win.col(p.col, start + q));
          S += (double)expf((float)(sc - m));
        }
        S = team_sum<T>(S, tmask);
        wr.m = m;
        wr.inv_s = (float)(1.0 / S);
        __syncwarp(tmask);
      }
    };
    float out[V];
    row_segments<V, G, false, R, XE>(p, win, wr, start, d, 0, (d + kSeg - 1) / kSeg, xb, nact, tl, sg, tmask,
                                 s_tc[team], s_tw[team], hl, kGat ? &s_cache[team][0] : nullptr, kGat ? kCache : 0,
                                 out, stats);
    finish_row<R, V>(out, d, p.mean);
    if (sg == 0 && active) epilogue<V>(p, r, col0, out, nvalid);
  }
  // no CTA may exit with bulk copies still writing its shared memory
  if (tid == 0) ensure(win.we);
}

// Host-side plan: vector width V from alignment, group width G from the slab
// width, row-block size C, and the slab-major grid.
struct EngineLaunch {
  int V, G;
  int64_t slab_cols, nslab, block_nnz, nblk;
};

gsp_status engine_plan(int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t f, int64_t head_dim, int vmax,
                       int32_t slab_req, int32_t block_req, EngineLaunch *L, int max_hpt);

// gat.cu: alpha = row softmax of the GAT scores (fp64 statistics)
gsp_status launch_row_softmax_scores(const gsp_csr *a, const float *el, const float *er, double slope, int H,
                                     float *alpha, cudaStream_t s);

// heads per team for a multi-head launch planned with slab L.slab_cols.  A
// team holds hpt > 1 heads only when the slab is exactly hpt whole heads of
// whole lanes (engine_plan's multi-head plan); a single head (whose plan is
// the plain one, possibly wider than d) or a slab inside a head gives 1.
inline int engine_hpt(const EngineLaunch &L, int64_t head_dim, int64_t heads) {
  if (heads <= 1 || head_dim <= 0 || L.slab_cols <= head_dim) return 1;
  if (L.slab_cols % head_dim || head_dim % L.V) return 1;
  const int64_t hpt = L.slab_cols / head_dim;
  if (hpt > heads || hpt > kMaxHpt || L.G % hpt) return 1;
  return (int)hpt;
}

// y may take the V-wide (at most float4) stores
inline int engine_y_vec_ok(const EngineLaunch &L, const float *y, int64_t ldy) {
  const int vw = L.V == 8 ? 4 : L.V;
  return (ldy % vw == 0) && ((reinterpret_cast<uintptr_t>(y) % (4 * vw)) == 0);
}

// 32-bit gather offsets: row c of x starts at vector c * ldxv.
inline gsp_status engine_ldxv(EngineParams &p, const EngineLaunch &L, int64_t n_cols, int64_t ldx) {
  const int64_t ldxv = ldx / (L.V == 8 ? 4 : L.V);
  if (n_cols > 0 && (n_cols - 1) * ldxv + ldxv >= (int64_t(1) << 32))
    return fail(GSP_ERR_UNSUPPORTED, "feature matrix too large for 32-bit vector offsets");
  p.ldxv = (uint32_t)ldxv;
  return GSP_OK;
}

// Fill the CSR-window staging fields of p: col (and val, if given) are
// staged through shared memory by TMA when 16-byte aligned.
inline void engine_stage(EngineParams &p, const EngineLaunch &L, int64_t nnz, const int32_t *col, const float *val) {
  p.nnz = nnz;
  p.stage = (nnz > 0 && aligned16(col)) ? 1 : 0;
  p.stage_val = (p.stage && val && aligned16(val)) ? val : nullptr;
  p.win_cap = (int)(((L.block_nnz + kHub + 8) + 3) & ~int64_t(3));
  p.stage_hm = nullptr;
  p.stage_hm_stride = 0;
  p.stage_heads = 0;
  p.mean = 0;
  p.hpt = 1;
  p.acc = nullptr;
  p.acc_src = nullptr;
  p.ldacc = p.ldsrc = 0;
  p.acc_coef = p.src_coef = 0.0f;
  p.skip_y = p.acc_vec_ok = p.src_vec_ok = 0;
  p.bias = nullptr;
  p.act = 0;
}

template <int V, int G, class W, class R, class XE = XF32<V>>
gsp_status engine_launch_vg(const EngineLaunch &L, const EngineParams &p, const W &w, cudaStream_t s) {
  const int64_t grid = L.nslab * L.nblk;
  if (grid <= 0) return GSP_OK;
  if (grid >= (int64_t(1) << 31)) return fail(GSP_ERR_UNSUPPORTED, "grid too large (%lld CTAs)", (long long)grid);
  const size_t smem =
      p.stage ? (size_t)p.win_cap * 4 * ((p.stage_val ? 2 : 1) + (p.stage_hm ? p.stage_heads : 0)) : 0;
  if (smem > 0) {  // static + dynamic may exceed the 48 KB default: raise the cap once per device
    static std::atomic<int> granted[64];  // per device: largest dynamic smem already granted
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || granted[dev].load(std::memory_order_relaxed) < (int)smem) {
      if (cudaFuncSetAttribute(engine_kernel<V, G, W, R, XE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
        return check_launch("cudaFuncSetAttribute(engine_kernel)");
      if (dev >= 0 && dev < 64) granted[dev].store((int)smem, std::memory_order_relaxed);
    }
  }
  engine_kernel<V, G, W, R, XE><<<(unsigned)grid, kThreads, smem, s>>>(p, w);
  return check_launch("engine_kernel");
}

template <int V, class W, class R>
gsp_status engine_launch_v(const EngineLaunch &L, const EngineParams &p, const W &w, cudaStream_t s) {
  switch (L.G) {
    case 1: return engine_launch_vg<V, 1, W, R>(L, p, w, s);
    case 2: return engine_launch_vg<V, 2, W, R>(L, p, w, s);
    case 4: return engine_launch_vg<V, 4, W, R>(L, p, w, s);
    case 8: return engine_launch_vg<V, 8, W, R>(L, p, w, s);
    case 16: return engine_launch_vg<V, 16, W, R>(L, p, w, s);
    case 32: return engine_launch_vg<V, 32, W, R>(L, p, w, s);
  }
  return fail(GSP_ERR_UNSUPPORTED, "bad group width %d", L.G);
}

template <class W, class R = RedSum>
gsp_status engine_launch(const EngineLaunch &L, const EngineParams &p, const W &w, cudaStream_t s) {
  switch (L.V) {
    case 8: return engine_launch_vg<8, 32, W, R>(L, p, w, s);
    case 4: return engine_launch_v<4, W, R>(L, p, w, s);
    case 2: return engine_launch_v<2, W, R>(L, p, w, s);
    case 1: return engine_launch_v<1, W, R>(L, p, w, s);
  }
  return fail(GSP_ERR_UNSUPPORTED, "bad vector width %d", L.V);
}

// fp16 feature storage (XF16): V = 8 halves per lane (16-byte loads) or 1
template <class W, class R = RedSum>
gsp_status engine_launch_f16(const EngineLaunch &L, const EngineParams &p, const W &w, cudaStream_t s) {
  if (L.V == 8) {
    switch (L.G) {
      case 1: return engine_launch_vg<8, 1, W, R, XF16<8>>(L, p, w, s);
      case 2: return engine_launch_vg<8, 2, W, R, XF16<8>>(L, p, w, s);
      case 4: return engine_launch_vg<8, 4, W, R, XF16<8>>(L, p, w, s);
      case 8: return engine_launch_vg<8, 8, W, R, XF16<8>>(L, p, w, s);
      case 16: return engine_launch_vg<8, 16, W, R, XF16<8>>(L, p, w, s);
      case 32: return engine_launch_vg<8, 32, W, R, XF16<8>>(L, p, w, s);
    }
  } else if (L.V == 4) {
    switch (L.G) {
      case 1: return engine_launch_vg<4, 1, W, R, XF16<4>>(L, p, w, s);
      case 2: return engine_launch_vg<4, 2, W, R, XF16<4>>(L, p, w, s);
      case 4: return engine_launch_vg<4, 4, W, R, XF16<4>>(L, p, w, s);
      case 8: return engine_launch_vg<4, 8, W, R, XF16<4>>(L, p, w, s);
      case 16: return engine_launch_vg<4, 16, W, R, XF16<4>>(L, p, w, s);
      case 32: return engine_launch_vg<4, 32, W, R, XF16<4>>(L, p, w, s);
    }
  } else if (L.V == 1) {
    switch (L.G) {
      case 1: return engine_launch_vg<1, 1, W, R, XF16<1>>(L, p, w, s);
      case 2: return engine_launch_vg<1, 2, W, R, XF16<1>>(L, p, w, s);
      case 4: return engine_launch_vg<1, 4, W, R, XF16<1>>(L, p, w, s);
      case 8: return engine_launch_vg<1, 8, W, R, XF16<1>>(L, p, w, s);
      case 16: return engine_launch_vg<1, 16, W, R, XF16<1>>(L, p, w, s);
      case 32: return engine_launch_vg<1, 32, W, R, XF16<1>>(L, p, w, s);
    }
  }
  return fail(GSP_ERR_UNSUPPORTED, "fp16 engine: bad V %d / G %d", L.V, L.G);
}

// Explicit instantiations live in engine_inst_*.cu (one TU per weight /
// reduce family, compiled in parallel); other TUs only declare them.
#define GSP_ENGINE_INSTANCES(X) \
  X(WeightVal, RedSum, sum)     \
  X(WeightOne, RedSum, sum)     \
  X(WeightVal, RedMax, maxmin)  \
  X(WeightOne, RedMax, maxmin)  \
  X(WeightVal, RedMin, maxmin)  \
  X(WeightOne, RedMin, maxmin)  \
  X(WeightAlpha, RedSum, alpha) \
  X(WeightAlphaHM, RedSum, alpha) \
  X(WeightGat, RedSum, gat)     \
  X(WeightGatPre, RedSum, gat)
#ifndef GSP_ENGINE_INSTANTIATE
extern template gsp_status engine_launch_f16<WeightVal, RedSum>(const EngineLaunch &, const EngineParams &,
                                                               const WeightVal &, cudaStream_t);
extern template gsp_status engine_launch_f16<WeightOne, RedSum>(const EngineLaunch &, const EngineParams &,
                                                               const WeightOne &, cudaStream_t);
#define GSP_ENGINE_EXTERN(W, R, tu) \
  extern template gsp_status engine_launch<W, R>(const EngineLaunch &, const EngineParams &, const W &, cudaStream_t);
GSP_ENGINE_INSTANCES(GSP_ENGINE_EXTERN)
#undef GSP_ENGINE_EXTERN
#endif

}  // namespace gsp
