/*
 * gsp.h -- C ABI of libgsp: B200-native (sm_100a) sparse GNN operators after
 * CogDL (arXiv 2103.00959), §4 "Efficiency of CogDL".
 *
 * Citations: "P:n" = PAPER.md line n, with the section / equation named;
 * "S:n" = SPEC.md line n (interface source only); "A<k>" = reading k of the
 * ambiguity register in DESIGN.md.
 *
 * CONVENTIONS (apply to every call)
 *  - Memory.  Every array argument is caller-owned DEVICE memory unless the
 *    parameter says "host".  The library never allocates device memory; calls
 *    that need scratch take a caller workspace sized by a *_workspace query.
 *  - Streams.  Every call enqueues its kernels on `stream` (a cudaStream_t;
 *    NULL = legacy default stream) and returns without synchronising, except
 *    gsp_coo_to_csr and (with a host output) gsp_partition_rows, which
 *    synchronise `stream`
 *    (documented on each).
 *  - Layout.  Dense matrices are row-major fp32 with an explicit row stride
 *    `ld` in elements (ld >= width).  Multi-head matrices are [n][H][D]
 *    (D fastest, A14); per-edge per-head arrays are [nnz][H] in canonical CSR
 *    order (edge-major, head-minor).  Vectorised (16-byte) paths are
 *    used when ld % 4 == 0 and base pointers are 16-byte aligned; otherwise a
 *    narrower path runs.  Misalignment is never an error.
 *  - Outputs are fully overwritten (beta = 0); empty rows give zeros.
 *    Columns of an output beyond its logical width (the ld padding) are not
 *    written.
 *  - Errors.  Arguments are validated on the host BEFORE any launch; on a
 *    host-detected error the call returns non-zero and touches nothing.
 *    gsp_last_error_detail() returns a thread-local description of the last
 *    error.  Launch failures return GSP_ERR_CUDA.
 *  - Determinism.  Every call is bitwise reproducible run to run (no
 *    floating-point atomics).  gsp_spmm / gsp_multihead_spmm /
 *    gsp_gat_aggregate use a summation order that depends only on the row
 *    (DESIGN.md §Summation order), so the result of a row does not depend on
 *    which other rows are in the call: a row-partitioned multi-GPU run is
 *    bitwise equal to the single-GPU run.
 *  - Threads.  Re-entrant; no global mutable state except the thread-local
 *    error string, the thread-local flags of gsp_set_flags and a per-device
 *    cached SM count.
 */
#ifndef GSP_H_
#define GSP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSP_VERSION 2

/* ABI-compatible with cudaStream_t / CUstream. */
typedef struct CUstream_st *gsp_stream;

typedef enum {
  GSP_OK = 0,
  GSP_ERR_INVALID_ARG = 1,     /* null pointer, negative size, ld < width, ... */
  GSP_ERR_INDEX_RANGE = 2,     /* an edge endpoint outside [0, n)       */
  GSP_ERR_NEGATIVE_WEIGHT = 3, /* A_ij >= 0 violated                   */
  GSP_ERR_NONFINITE = 4,       /* NaN / Inf weight or (validate mode) logit    */
  GSP_ERR_ALIAS = 5,           /* input and output ranges overlap              */
  GSP_ERR_WORKSPACE = 6,       /* workspace missing or too small               */
  GSP_ERR_UNSUPPORTED = 7,     /* size beyond the supported range              */
  GSP_ERR_CUDA = 8             /* CUDA launch / runtime error                  */
} gsp_status;

typedef enum { GSP_I32 = 0, GSP_I64 = 1 } gsp_index_type;

/* flags: GSP_UNDIRECTED for gsp_coo_to_csr; GSP_VALIDATE for gsp_set_flags */
enum { GSP_UNDIRECTED = 1u, GSP_VALIDATE = 2u };

/* ---------------------------------------------------------------------------
 * Validate mode ("pre: all finite ... errors: non-finite
 * logit"; reading A12).  gsp_set_flags(GSP_VALIDATE) turns it on for calls
 * made BY THE CALLING THREAD (thread-local; 0 turns it off; other bits are
 * GSP_ERR_INVALID_ARG).  In validate mode gsp_edge_softmax checks `logits`,
 * and gsp_gat_aggregate, gsp_gat_aggregate_bias_act and
 * gsp_gat_aggregate_backward check `el` and `er`, for NaN / Inf before any
 * compute launch: one streaming kernel per array, then the call synchronises
 * its stream once and returns GSP_ERR_NONFINITE (outputs untouched) if any
 * value is non-finite.  Outside validate mode nothing is checked and a NaN
 * propagates within its row only.  Validating calls on one device are
 * serialised internally. */
gsp_status gsp_set_flags(uint32_t flags);
uint32_t gsp_get_flags(void);

/*
 * Borrowed view of a CSR matrix in device memory ("CogDL utilizes
 * CSR-format design").  Rows are sorted; within a row, columns are strictly
 * increasing (canonical form produced by gsp_coo_to_csr).
 *   n_rows   rows; n_cols columns (= n for a whole graph; for a slice made by
 *            gsp_csr_slice, the padded all-gathered row count P * rows_padded)
 *   nnz      stored entries; row_ptr[n_rows] == nnz
 *   row_ptr  int64 [n_rows + 1], row_ptr[0] == 0, nondecreasing
 *   col_idx  int32 [nnz], each < n_cols
 *   val      fp32 [nnz], or NULL meaning every weight is 1.0 (psi = copy)
 * n_rows, n_cols < 2^31.
 */
typedef struct {
  int64_t n_rows, n_cols, nnz;
  const int64_t *row_ptr;
  const int32_t *col_idx;
  const float *val;
} gsp_csr;

/* ---------------------------------------------------------------------------
 * a1. COO -> canonical CSR of A~ = A + fill * I.
 * P:625-632 (§4 Graph Notations: A binary or weighted, A_ij >= 0, directed or
 * undirected), P:244 (Eq. gcn_layer, A~ = A + I_n), P:646 (CSR design),
 * P:1707 (Graph(edge_index=...)).  Readings A2, A4, A5, A6.
 *
 * Input pair i is (src[i], dst[i]) with weight w[i] (w NULL => 1.0); it is
 * stored at row src[i], column dst[i] (A1).  With GSP_UNDIRECTED, (dst, src)
 * is also stored when src != dst.  If fill != 0, (u, u, fill) is added for
 * every u.  Duplicates (including an input self-loop plus the fill) are
 * coalesced by summing their weights in input order in fp64 and rounding once
 * to fp32; explicit zero weights stay in the structure.
 *
 *   n, m          nodes, input pairs (m >= 0, n >= 0, n < 2^31,
 *                 (2m + n) < 2^32)
 *   src, dst      device int32 or int64 (per `it`) [m]
 *   w             device fp32 [m] or NULL
 *   row_ptr       out, device int64 [n + 1]
 *   col_idx, val  out, device int32 / fp32 [nnz_max] (nnz_max from the query)
 *   nnz_out       out, HOST int64: number of stored entries
 *   ws, ws_bytes  device workspace, >= gsp_coo_to_csr_workspace()'s size
 * Errors: GSP_ERR_INDEX_RANGE, GSP_ERR_NEGATIVE_WEIGHT, GSP_ERR_NONFINITE are
 * detected on the device; the call synchronises `stream` once (to read
 * nnz and the validation flags).  On a device-detected error the outputs are
 * left unspecified (no out-of-bounds writes occur).
 */
gsp_status gsp_coo_to_csr_workspace(int64_t n, int64_t m, uint32_t flags, float fill,
                                    size_t *ws_bytes, int64_t *nnz_max);
gsp_status gsp_coo_to_csr(int64_t n, int64_t m, const void *src, const void *dst,
                          gsp_index_type it, const float *w, uint32_t flags, float fill,
                          int64_t *row_ptr, int32_t *col_idx, float *val, int64_t *nnz_out,
                          void *ws, size_t ws_bytes, gsp_stream stream);

/* ---------------------------------------------------------------------------
 * a2. Degree and GCN symmetric normalisation A^ = D~^-1/2 A~ D~^-1/2.
 * P:244 (Eq. gcn_layer: D~_ii = sum_j A~_ij).  Readings A3, A7, A8.
 *   d_u = sum of row u's weights, fp64 (exact whenever the row sum is exact
 *   in fp64, A8); val_out[e] = fp32( w_e / sqrt(d_u * d_v) ) with IEEE
 *   round-to-nearest double operations (bit-identical to the oracle), 0 when
 *   d_u * d_v == 0.  a->val must be non-NULL (the A~ weights).  val_out may
 *   equal a->val (in place).  Requires a square matrix (n_rows == n_cols).
 *   deg_out  device fp64 [n_rows] receiving d, or NULL;
 *   ws       when deg_out is NULL: device, 8-byte aligned, >=
 *            gsp_sym_normalize_workspace() bytes (holds d between the two
 *            passes; the library never allocates) -- else ignored (may be NULL).
 * Errors: GSP_ERR_WORKSPACE if deg_out and ws are both missing / too small;
 * GSP_ERR_ALIAS if val_out overlaps the degree array.
 */
gsp_status gsp_sym_normalize_workspace(const gsp_csr *a, size_t *ws_bytes);
gsp_status gsp_sym_normalize(const gsp_csr *a, float *val_out, double *deg_out, void *ws, size_t ws_bytes,
                             gsp_stream stream);

/* ---------------------------------------------------------------------------
 * a3. SpMM  Y = A X  (GSpMM, phi = sum, psi = multiply).
 * P:640-645 (§4.1 Eq. formula:1; "SpMM operator H^(l+1) <- A H^(l)"),
 * P:646-648 (kernel design: CSR, coalesced feature access, cached indices).
 *   x  device fp32 [a->n_cols][ldx], columns [0, f) used; the whole
 *      [n_cols][ldx] extent must be readable: padding columns [f, ldx) that
 *      share a 16-byte vector with column f-1 may be read, their values are
 *      never used (any bits, including NaN, are fine)
 *   y  device fp32 [a->n_rows][ldy], columns [0, f) written
 *   f >= 0, ldx >= f, ldy >= f.  x and y must not overlap (GSP_ERR_ALIAS).
 * fp32 multiply-add; error bound per element in DESIGN.md §Summation order
 * (|y - y_exact| <= ~100 u * sum_j |a_ij x_jk| for rows up to 1.5M entries).
 */
gsp_status gsp_spmm(const gsp_csr *a, const float *x, int64_t f, int64_t ldx, float *y,
                    int64_t ldy, gsp_stream stream);

/* gsp_spmm_ex with slab_cols == 256 reads two float4 per lane: it needs
 * ldx % 8 == 0 and a 32-byte aligned x (else GSP_ERR_INVALID_ARG). */

/* gsp_spmm_f16: gsp_spmm with fp16 feature storage (mixed
 * precision "fp16=True"): x device IEEE binary16 [a->n_cols][ldx] (padding as
 * for gsp_spmm), y device fp32 [a->n_rows][ldy].  Every x value is converted
 * exactly to fp32; products and sums are fp32 in the same order as gsp_spmm,
 * so the error bound is gsp_spmm's with x replaced by its fp16 values.  8-byte
 * gathers of 4 halves when ldx % 4 == 0 and x is 8-byte aligned (scalar
 * otherwise). */
gsp_status gsp_spmm_f16(const gsp_csr *a, const void *x, int64_t f, int64_t ldx, float *y, int64_t ldy,
                        gsp_stream stream);

/* ---------------------------------------------------------------------------
 * GSpMM with a selectable reduce operator phi (NEXT-2).
 * P:640-646 (§4.1 Eq. formula:1, "users could choose the reduce or compute
 * operator"), P:648 ("min and max as reduce functions"), P:1355 (Fig. gspmm:
 * "mean and sum as reduce functions").  psi is multiply by a->val, or copy
 * when a->val is NULL.  y[u,k] = phi over row u of psi(x[col_e,k], val_e):
 *   GSP_REDUCE_SUM   sum (== gsp_spmm)
 *   GSP_REDUCE_MEAN  sum / (number of entries in row u)
 *   GSP_REDUCE_MAX / GSP_REDUCE_MIN  row-wise extremum; exact (no rounding
 *                    beyond the fp32 product), so bit-identical to any order
 * Empty rows give 0 for every operator.  Arguments as gsp_spmm. */
typedef enum { GSP_REDUCE_SUM = 0, GSP_REDUCE_MEAN = 1, GSP_REDUCE_MAX = 2, GSP_REDUCE_MIN = 3 } gsp_reduce;
gsp_status gsp_gspmm(const gsp_csr *a, gsp_reduce reduce, const float *x, int64_t f, int64_t ldx, float *y,
                     int64_t ldy, gsp_stream stream);

/* ---------------------------------------------------------------------------
 * K-step propagation (NEXT-4): y = sum_{k=0..K} theta_k A^k x.
 * P:297 (graph diffusion A_bar = sum_i alpha_i A^i), P:255 (APPNP, personalized
 * PageRank: theta_k = alpha (1 - alpha)^k), P:282 (SGC: theta = e_K);
 * S:171-188.  K >= 1 launches of the SpMM engine with a fused accumulate
 * epilogue; step 1 folds theta_0 x in, so no separate scale pass.
 *   theta  HOST fp64 [K+1]
 *   ws     device workspace of gsp_propagate_workspace() bytes (the t_k
 *          ping-pong buffers; 0 for K == 1)
 * A must be square; x and y must not overlap.
 *
 * gsp_spmm_accumulate is one step with the fused epilogue:
 *   t = A x                        (written to t unless t == NULL)
 *   acc = coef * t + (src != NULL ? src_coef * src : acc)      (fp32 fma)
 * It is the building block of the row-partitioned multi-GPU propagation
 * (A may be a rectangular slice there: x has n_cols rows, t/acc/src n_rows). */
gsp_status gsp_spmm_accumulate(const gsp_csr *a, const float *x, int64_t f, int64_t ldx, float *t, int64_t ldt,
                               float *acc, int64_t ldacc, float coef, const float *src, int64_t ldsrc,
                               float src_coef, gsp_stream stream);
gsp_status gsp_propagate_workspace(const gsp_csr *a, int64_t f, int64_t K, size_t *ws_bytes);
gsp_status gsp_propagate(const gsp_csr *a, const float *x, int64_t f, int64_t ldx, int64_t K, const double *theta,
                         float *y, int64_t ldy, void *ws, size_t ws_bytes, gsp_stream stream);

/* Tuning knobs for gsp_spmm_ex (0 = automatic).  Results are bitwise
 * identical for every setting (the summation order does not depend on them). */
typedef struct {
  int32_t slab_cols;   /* columns per slab: 0 = auto (L2-resident slab), else 16..512 */
  int32_t block_nnz;   /* nonzeros per CTA row block: 0 = auto                          */
  int32_t reserved[6];
} gsp_spmm_opts;
gsp_status gsp_spmm_ex(const gsp_csr *a, const float *x, int64_t f, int64_t ldx, float *y,
                       int64_t ldy, const gsp_spmm_opts *opts, gsp_stream stream);

/* The launch plan gsp_spmm / gsp_spmm_ex(opts) would use for these arguments
 * (host only, no launch): number of kernel launches (1, or 2 when a narrower
 * tail launch covers the last columns), the main slab width and the tail slab
 * width (0 if none).  Any output pointer may be NULL. */
gsp_status gsp_spmm_plan_info(const gsp_csr *a, const float *x, int64_t f, int64_t ldx,
                              const gsp_spmm_opts *opts, int32_t *launches, int32_t *slab_cols,
                              int32_t *tail_slab_cols);

/* ---------------------------------------------------------------------------
 * a6. Edge-wise softmax per head, max-subtracted.
 * P:653-656 (§4.1: alpha'_uv = exp(alpha_uv) / sum_{w in N(u)} exp(alpha_uw);
 * "find the max value ... subtract ... exponent ... reduce ... the sum").
 * Readings A9, A10, A12.
 *   logits, alpha  device fp32 [nnz][heads]; alpha may equal logits (in place)
 *   heads >= 1.  Empty rows emit nothing.  s - max is formed in fp64 before the
 *   fp32 exponential; the row sum is accumulated in fp64.
 */
gsp_status gsp_edge_softmax(const gsp_csr *a, int32_t heads, const float *logits, float *alpha,
                            gsp_stream stream);

/* ---------------------------------------------------------------------------
 * a7. Multi-head SpMM: Y[u,h,:] = sum_{e in row u} alpha[e,h] * Z[col_e,h,:].
 * P:648-649 (§4.1 multi-head SpMM; heads share the sparsity pattern), A14.
 *   alpha  device fp32 [nnz][heads]
 *   z      device fp32 [a->n_cols][ldz], viewed as [H][D]; ldz >= heads*d
 *   y      device fp32 [a->n_rows][ldy]; ldy >= heads*d; must not overlap z
 */
gsp_status gsp_multihead_spmm(const gsp_csr *a, int32_t heads, const float *alpha,
                              const float *z, int64_t d, int64_t ldz, float *y, int64_t ldy,
                              gsp_stream stream);

/* ---------------------------------------------------------------------------
 * a4. GAT attention projection (split form of a^T [z_u || z_v], A13):
 *   el[u,h] = sum_d a_l[h,d] z[u,h,d],  er[u,h] = sum_d a_r[h,d] z[u,h,d].
 *   z device fp32 [n][ldz]; a_l, a_r device fp32 [heads][d];
 *   el, er device fp32 [n][heads].
 */
gsp_status gsp_attn_project(int64_t n, int32_t heads, int64_t d, const float *z, int64_t ldz,
                            const float *a_l, const float *a_r, float *el, float *er,
                            gsp_stream stream);

/* ---------------------------------------------------------------------------
 * a5 + a6 + a7 fused.  GAT aggregation (P:253 GAT):
 *   s[e,h]  = LeakyReLU(el[u,h] + er[v,h]; negative_slope)     e = (u,v), A13
 *   alpha   = edge softmax of s over row u, per head
 *   Y[u,h,:] = sum_e alpha[e,h] Z[v,h,:]
 * Three schedules, same result up to fp rounding of the statistics, chosen
 * by the workspace (16-byte aligned; heads | 32 for the first two):
 *  - ws >= gsp_gat_workspace bytes (128-byte aligned) and alpha_out NULL:
 *    "staged".  A statistics launch (lane per (row, head); long rows as
 *    per-warp partials merged in warp order) writes alpha HEAD-MAJOR
 *    into ws ([H][round_up(nnz, 32)] fp32); the aggregate launch stages the
 *    alpha runs of its slab's heads with the CSR window (TMA bulk copies) and
 *    gathers Z with weights read from shared memory;
 *  - ws >= n_rows * heads * 16 bytes (or alpha_out requested): the statistics
 *    launch writes (m, 1/S) per (row, head) and the aggregate forms alpha on
 *    the fly (several whole heads per team);
 *  - ws NULL (or too small): ONE launch; the team that owns a (row, head)
 *    first reduces the row's statistics (hub rows: the whole CTA) and then
 *    runs the fused score -> softmax -> aggregate pass.
 * Per-edge messages (alpha * Z rows) are never materialised; per-edge alpha
 * only in the staged schedule's workspace or when alpha_out is non-NULL.
 *   el  device fp32 [a->n_rows][heads];  er device fp32 [a->n_cols][heads]
 *   z   device fp32 [a->n_cols][ldz] ([H][D]);  y device fp32 [a->n_rows][ldy]
 *   alpha_out  device fp32 [nnz][heads] or NULL
 *   ws  NULL, or device workspace of up to gsp_gat_workspace(a, heads) bytes
 *       (= max(n_rows * heads * 16, heads * round_up(nnz, 32) * 4))
 * The score is formed in fp64 (el + er, slope multiply, minus the row max) and
 * rounded once before the fp32 exponential.
 */
gsp_status gsp_gat_workspace(const gsp_csr *a, int32_t heads, size_t *ws_bytes);
gsp_status gsp_gat_aggregate(const gsp_csr *a, int32_t heads, const float *el, const float *er,
                             double negative_slope, const float *z, int64_t d, int64_t ldz,
                             float *y, int64_t ldy, float *alpha_out, void *ws, size_t ws_bytes,
                             gsp_stream stream);

/* ---------------------------------------------------------------------------
 * NEXT-3: GAT backward.  P:652 (§4.1: SDDMM T = A (.) (P Q^T) "is used for
 * back-propagating the gradients to the sparse adjacency matrix since the
 * adjacency matrix of the GAT model is computed by the attention mechanism"),
 * P:653-656 (edge softmax).
 *
 * gsp_csr_transpose: A^T in canonical form (n_cols rows) and perm[e'] = the
 *   index in A of entry e' of A^T (so per-entry arrays of A can be read in A^T
 *   order).  Outputs: row_ptr_t int64 [n_cols+1], col_t int32 [nnz],
 *   perm int32 [nnz]; nnz < 2^31; ws >= gsp_csr_transpose_workspace bytes,
 *   256-byte aligned.  Bit-exact (integer work).
 * gsp_sddmm: out[e,h] = sum_k p[u,h,k] q[v,h,k] for e = (u,v) (structural:
 *   A's values are not multiplied in).  p [n_rows][ldp], q [n_cols][ldq]
 *   viewed as [H][D]; out fp32 [nnz][H].
 * gsp_edge_softmax_backward: ds = alpha (dalpha - sum_row alpha dalpha) per
 *   head (fp64 row dot); heads must divide 32.  ds may equal dalpha.
 * gsp_gat_aggregate_backward: given dY of gsp_gat_aggregate (same a, el, er,
 *   z, slope), writes dz [n][lddz] (= A^T_alpha dY, overwritten),
 *   d_el [n][H] and d_er [n][H] (the LeakyReLU-score gradients; the score's
 *   dependence on Z goes through gsp_attn_project_backward).  at/perm from
 *   gsp_csr_transpose(a).  alpha is recomputed from el, er.  ws >=
 *   gsp_gat_backward_workspace bytes.  Launches: softmax, SDDMM, fused
 *   softmax/LeakyReLU backward with row sums, column sums, A^T SpMM.
 * gsp_attn_project_backward: dz[u,h,:] += d_el[u,h] a_l[h,:] + d_er[u,h] a_r[h,:];
 *   d_al[h,:] = sum_u d_el[u,h] z[u,h,:], d_ar likewise (fixed-order
 *   reduction, fp64 partials in ws >= gsp_attn_project_backward_workspace). */
gsp_status gsp_csr_transpose_workspace(const gsp_csr *a, size_t *ws_bytes);
gsp_status gsp_csr_transpose(const gsp_csr *a, int64_t *row_ptr_t, int32_t *col_t, int32_t *perm, void *ws,
                             size_t ws_bytes, gsp_stream stream);
gsp_status gsp_sddmm(const gsp_csr *a, int32_t heads, const float *p, int64_t d, int64_t ldp, const float *q,
                     int64_t ldq, float *out, gsp_stream stream);
gsp_status gsp_edge_softmax_backward(const gsp_csr *a, int32_t heads, const float *alpha, const float *dalpha,
                                     float *ds, gsp_stream stream);
gsp_status gsp_gat_backward_workspace(const gsp_csr *a, int32_t heads, size_t *ws_bytes);
gsp_status gsp_gat_aggregate_backward(const gsp_csr *a, const gsp_csr *at, const int32_t *perm, int32_t heads,
                                      const float *el, const float *er, double negative_slope, const float *z,
                                      int64_t d, int64_t ldz, const float *dy, int64_t lddy, float *dz,
                                      int64_t lddz, float *d_el, float *d_er, void *ws, size_t ws_bytes,
                                      gsp_stream stream);
gsp_status gsp_attn_project_backward_workspace(int64_t n, int32_t heads, int64_t d, size_t *ws_bytes);
gsp_status gsp_attn_project_backward(int64_t n, int32_t heads, int64_t d, const float *z, int64_t ldz,
                                     const float *a_l, const float *a_r, const float *d_el, const float *d_er,
                                     float *dz, int64_t lddz, float *d_al, float *d_ar, void *ws, size_t ws_bytes,
                                     gsp_stream stream);

/* ---------------------------------------------------------------------------
 * NEXT-1: layers for 2-layer GCN / GAT inference (P:239-246 Eq. gcn_layer
 * H^(l+1) = sigma(A^ H^(l) W^(l)); P:661-663 Table spmm_time).
 * gsp_linear: row-major y[n][f_out] = x[n][f_in] w[f_in][f_out] (ldw >= f_out).
 *   With ws >= gsp_linear_workspace(f_in, f_out) bytes (device, any
 *   alignment), f_out <= 4096, ldx % 4 == 0 and x 16-byte aligned: tcgen05
 *   tensor cores, kind::tf32 with 3xTF32 splitting (x = hi + lo with hi the
 *   MMA's truncated read of the raw fp32 x, w = hi + lo pre-split by
 *   rounding; x w ~= lo.hi + hi.lo + hi.hi, fp32 accumulation in TMEM;
 *   per-product error <= 2^-19 |x||w|), operands staged by TMA (SWIZZLE_64B: 16-float K
 *   tiles), one CTA per (128 rows, <= 256 output columns); for f_out <= 128
 *   and f_in >= 384 two adjacent row tiles run as a cluster (CTA pair) that
 *   shares the W tiles by TMA multicast (needs cluster launch support, every
 *   B200).  Results do not depend on the tiling.  Otherwise (ws
 *   NULL / too small, wider or unaligned operands) a
 *   cuBLAS SGEMM with fp32 compute (no TF32); one cuBLAS handle per (thread,
 *   device) is created on first use.
 * gsp_spmm_bias_act: y = act(A x + bias) with bias [f] (nullable) and the
 *   activation fused into the SpMM epilogue.
 * gsp_gcn_layer: y = act(A (x w) + bias): gsp_linear into ws, then
 *   gsp_spmm_bias_act.  Every argument (act, pointers, leading dimensions, y
 *   and x against ws: GSP_ERR_ALIAS) is checked before the first enqueue.  ws >= gsp_gcn_layer_workspace(a->n_cols, f_in, f_out)
 *   (holds x w and the tensor-core GEMM's split-W workspace).
 * gsp_gat_aggregate_bias_act: gsp_gat_aggregate with y = act(Y + bias[H*D])
 *   fused (ELU for hidden GAT layers); ws as for gsp_gat_aggregate. */
typedef enum { GSP_ACT_NONE = 0, GSP_ACT_RELU = 1, GSP_ACT_ELU = 2 } gsp_act;
gsp_status gsp_linear_workspace(int64_t f_in, int64_t f_out, size_t *ws_bytes);
gsp_status gsp_linear(int64_t n, int64_t f_in, const float *x, int64_t ldx, const float *w, int64_t ldw,
                      int64_t f_out, float *y, int64_t ldy, void *ws, size_t ws_bytes, gsp_stream stream);
gsp_status gsp_spmm_bias_act(const gsp_csr *a, const float *x, int64_t f, int64_t ldx, const float *bias,
                             gsp_act act, float *y, int64_t ldy, gsp_stream stream);
gsp_status gsp_gcn_layer_workspace(int64_t n, int64_t f_in, int64_t f_out, size_t *ws_bytes);
gsp_status gsp_gcn_layer(const gsp_csr *a, const float *x, int64_t f_in, int64_t ldx, const float *w,
                         int64_t f_out, const float *bias, gsp_act act, float *y, int64_t ldy, void *ws,
                         size_t ws_bytes, gsp_stream stream);
gsp_status gsp_gat_aggregate_bias_act(const gsp_csr *a, int32_t heads, const float *el, const float *er,
                                      double negative_slope, const float *z, int64_t d, int64_t ldz,
                                      const float *bias, gsp_act act, float *y, int64_t ldy, void *ws,
                                      size_t ws_bytes, gsp_stream stream);

/* ---------------------------------------------------------------------------
 * Multi-GPU row partition.
 * gsp_partition_rows: row_bounds[p] = first row r with row_ptr[r] >=
 *   ceil(p * nnz / parts) for 0 < p < parts; row_bounds[0] = 0,
 *   row_bounds[parts] = n_rows; 1 <= parts <= 128.  Written to
 *   row_bounds_dev (DEVICE int64 [parts + 1]) and, when row_bounds_host
 *   (HOST int64 [parts + 1]) is non-NULL, copied there -- in that case the
 *   call synchronises `stream`.
 * gsp_csr_slice: the rows [row_bounds[rank], row_bounds[rank+1]) of `a`, with
 *   column c (owned by rank q: row_bounds[q] <= c < row_bounds[q+1]) remapped
 *   to q * rows_padded + (c - row_bounds[q]) -- its row in the buffer produced
 *   by an equal-count all-gather of per-rank feature shards padded to
 *   rows_padded rows.  row_bounds is HOST [parts + 1]; rows_padded >= the
 *   largest part.  Outputs (device): row_ptr_out int64 [rows + 1] (starts at
 *   0), col_out int32 [slice nnz], val_out fp32 [slice nnz] (NULL to skip;
 *   ignored when a->val is NULL).
 */
/* ---------------------------------------------------------------------------
 * Column blocks of A for an L2-sized X footprint (a3):
 * A = sum_k A_k with A_k the entries of A whose column lies in
 * [col_bounds[k], col_bounds[k+1]); Y = A X is then computed as
 * Y = A_0 X, Y += A_1 X, ... so each launch gathers from n_cols / blocks rows
 * of X (C4: a 60 MB instead of a 119 MB slab footprint per 128 columns).
 * gsp_csr_colblock_workspace: bytes of ws for `blocks` (1..8) blocks of a.
 * gsp_csr_colblock: col_bounds HOST [blocks + 1], nondecreasing, col_bounds[0]
 *   == 0, col_bounds[blocks] == n_cols.  Builds the blocks inside ws (device,
 *   caller-owned, >= gsp_csr_colblock_workspace bytes; any alignment) and
 *   fills the HOST array out[blocks] with CSRs that point into ws (valid as
 *   long as ws is); each block keeps the row order and the column order of
 *   a.  One stream sync (reads the block sizes).  A one-off per graph, like
 *   gsp_coo_to_csr.
 * gsp_spmm_blocked: y[:, :f] = sum_k blocks[k] x, summed in block order
 *   (block 0 writes y, block k adds its partial with one rounding): a fixed
 *   order per row, within the SpMM bound of gsp_spmm (one extra rounding per
 *   block); blocks must share n_rows / n_cols.  x, y as for gsp_spmm.
 */
gsp_status gsp_csr_colblock_workspace(const gsp_csr *a, int32_t blocks, size_t *ws_bytes);
gsp_status gsp_csr_colblock(const gsp_csr *a, const int64_t *col_bounds, int32_t blocks, void *ws, size_t ws_bytes,
                            gsp_csr *out, gsp_stream stream);
gsp_status gsp_spmm_blocked(const gsp_csr *blocks, int32_t nblocks, const float *x, int64_t f, int64_t ldx, float *y,
                            int64_t ldy, gsp_stream stream);

gsp_status gsp_partition_rows(const gsp_csr *a, int32_t parts, int64_t *row_bounds_dev,
                              int64_t *row_bounds_host, gsp_stream stream);
gsp_status gsp_csr_slice(const gsp_csr *a, const int64_t *row_bounds, int32_t parts, int32_t rank,
                         int64_t rows_padded, int64_t *row_ptr_out, int32_t *col_out,
                         float *val_out, gsp_stream stream);

/* ---------------------------------------------------------------------------
 * Misc. */
const char *gsp_status_string(gsp_status st);
const char *gsp_last_error_detail(void); /* thread-local; "" when none */
int gsp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GSP_H_ */
