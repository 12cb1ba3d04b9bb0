/*
 * oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the CogDL
 * (arXiv 2103.00959) sparse-operator hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2103_00959_b200/csrc, include/gsp.h) and includes neither.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared
 *        (IEEE double on x86-64 SSE2, no FMA contraction).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section / equation in
 * brackets); "S:n" = SPEC.md line n; "A<k>" = DESIGN.md ambiguity reading k.
 *
 * Every function works on caller-owned host arrays and returns 0 on success
 * or a negative code on invalid input.  Row-range entry points ([r0, r1))
 * write output row u at (u - r0) so huge graphs can be checked in pieces.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_ARG (-1)
#define ORC_ERR_RANGE (-2)
#define ORC_ERR_NEGATIVE (-3)
#define ORC_ERR_NONFINITE (-4)
#define ORC_ERR_CAPACITY (-5)
#define ORC_ERR_NOMEM (-6)

int orc_version(void) { return 1; }

/* ---------------------------------------------------------------------------
 * 1. COO -> canonical CSR of A~ = A + fill*I.
 *    P:625-632 [§4 Graph Notations: A binary or weighted, A_ij >= 0, directed
 *    or undirected; undirected => e_ij = e_ji, A_ij = A_ji];
 *    P:244 [Eq. gcn_layer: A~ = A + I_n]; P:646 [§4.1: CSR-format design];
 *    A2 (fill is ADDED to an existing (u,u)), A4 (duplicates summed in input
 *    order), A5 (undirected: (v,u) added for u != v), A6 (reject w < 0 and
 *    non-finite w; keep explicit zeros).
 *
 *    Entry i of the input (u_i, v_i, w_i) produces (u_i, v_i, w_i, pos=2i) and,
 *    when undirected and u_i != v_i, (v_i, u_i, w_i, pos=2i+1).  Node u's
 *    self-loop (fill != 0) is (u, u, fill, pos=2m+u).  Entries are sorted by
 *    (row, col, pos); equal (row, col) are summed in pos order in fp64 and
 *    rounded once to fp32.  row_ptr[u] = number of distinct entries in rows < u.
 * ------------------------------------------------------------------------- */
typedef struct {
  int64_t row, col, pos;
  double w;
} orc_entry;

static int cmp_entry(const void *pa, const void *pb) {
  const orc_entry *a = (const orc_entry *)pa, *b = (const orc_entry *)pb;
  if (a->row != b->row) return a->row < b->row ? -1 : 1;
  if (a->col != b->col) return a->col < b->col ? -1 : 1;
  if (a->pos != b->pos) return a->pos < b->pos ? -1 : 1;
  return 0;
}

int orc_build_csr(int64_t n, int64_t m, const int64_t *src, const int64_t *dst,
                  const float *w /* nullable: all 1.0 */, int undirected, float fill,
                  int64_t *row_ptr /* [n+1] */, int32_t *col /* [cap] */,
                  float *val /* [cap] */, int64_t cap, int64_t *nnz_out) {
  if (n < 0 || m < 0 || !row_ptr || !nnz_out || (m > 0 && (!src || !dst))) return ORC_ERR_ARG;
  int64_t total = 0;
  for (int64_t i = 0; i < m; ++i) {
    if (src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n) return ORC_ERR_RANGE;
    if (w) {
      if (!isfinite(w[i])) return ORC_ERR_NONFINITE;
      if (w[i] < 0.0f) return ORC_ERR_NEGATIVE;
    }
    total += (undirected && src[i] != dst[i]) ? 2 : 1;
  }
  if (!isfinite(fill)) return ORC_ERR_NONFINITE;
  if (fill < 0.0f) return ORC_ERR_NEGATIVE;
  if (fill != 0.0f) total += n;

  orc_entry *e = (orc_entry *)malloc(sizeof(orc_entry) * (size_t)(total > 0 ? total : 1));
  if (!e) return ORC_ERR_NOMEM;
  int64_t k = 0;
  for (int64_t i = 0; i < m; ++i) {
    double wi = w ? (double)w[i] : 1.0;
    e[k].row = src[i]; e[k].col = dst[i]; e[k].pos = 2 * i; e[k].w = wi; ++k;
    if (undirected && src[i] != dst[i]) {
      e[k].row = dst[i]; e[k].col = src[i]; e[k].pos = 2 * i + 1; e[k].w = wi; ++k;
    }
  }
  if (fill != 0.0f)
    for (int64_t u = 0; u < n; ++u) {
      e[k].row = u; e[k].col = u; e[k].pos = 2 * m + u; e[k].w = (double)fill; ++k;
    }
  qsort(e, (size_t)total, sizeof(orc_entry), cmp_entry);

  /* coalesce equal (row, col): fp64 sum in pos order, then one rounding */
  int64_t nnz = 0;
  for (int64_t u = 0; u <= n; ++u) row_ptr[u] = 0;
  for (int64_t a = 0; a < total;) {
    int64_t b = a;
    double s = 0.0;
    while (b < total && e[b].row == e[a].row && e[b].col == e[a].col) { s += e[b].w; ++b; }
    if (nnz >= cap) { free(e); return ORC_ERR_CAPACITY; }
    if (col) col[nnz] = (int32_t)e[a].col;
    if (val) val[nnz] = (float)s;
    row_ptr[e[a].row + 1] += 1;
    ++nnz;
    a = b;
  }
  for (int64_t u = 0; u < n; ++u) row_ptr[u + 1] += row_ptr[u];
  *nnz_out = nnz;
  free(e);
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * 2. Degree and symmetric normalisation.
 *    P:244 [Eq. gcn_layer: A^ = D~^-1/2 A~ D~^-1/2, D~_ii = sum_j A~_ij];
 *    A3 (row sums on both sides), A7 (a^ = 0 when d_u*d_v = 0), A8 (formula
 *    a^_uv = w_uv / sqrt(d_u * d_v), IEEE double, then one rounding to fp32).
 *    d_u is summed sequentially in column order.
 *    Outputs: deg [n] (nullable), a64 [nnz] (nullable, unrounded),
 *    a32 [nnz] (nullable, fp32-rounded a64).
 * ------------------------------------------------------------------------- */
int orc_sym_norm(int64_t n, const int64_t *row_ptr, const int32_t *col, const float *w,
                 double *deg, double *a64, float *a32) {
  if (n < 0 || !row_ptr || !col || !w) return ORC_ERR_ARG;
  double *d = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  if (!d) return ORC_ERR_NOMEM;
  for (int64_t u = 0; u < n; ++u) {
    double s = 0.0;
    for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) s += (double)w[e];
    d[u] = s;
    if (deg) deg[u] = s;
  }
  for (int64_t u = 0; u < n; ++u)
    for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
      double p = d[u] * d[col[e]];
      double r = 0.0;
      if (p != 0.0) {
        double q = sqrt(p);
        r = (double)w[e] / q;
      }
      if (a64) a64[e] = r;
      if (a32) a32[e] = (float)r;
    }
  free(d);
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * 3. SpMM  Y = A X  (GSpMM with phi = sum, psi = multiply).
 *    P:640-645 [§4.1 Eq. formula:1: h_u = phi(psi(h_v, h_e)), v in N(u),
 *    e = (u,v); "SpMM operator H^(l+1) <- A H^(l)"]; A1 (pair (u,v) is stored
 *    at row u, col v).  a == NULL means unit weights (psi = copy).
 *    y[u,k] = sum_e a_e * x[col_e, k] in fp64; cond[u,k] = sum_e |a_e x[col_e,k]|
 *    (the condition sum used by the parity bound).  Rows [r0, r1).
 * ------------------------------------------------------------------------- */
int orc_spmm(int64_t r0, int64_t r1, const int64_t *row_ptr, const int32_t *col,
             const double *a, const float *x, int64_t f, int64_t ldx,
             double *y, double *cond, int64_t ldy) {
  if (r0 < 0 || r1 < r0 || f < 0 || ldx < f || ldy < f || !row_ptr || (!col && r1 > r0) || !x || !y)
    return ORC_ERR_ARG;
  /* rows are independent: liboracle_omp.so (-fopenmp) runs them on all host
   * cores with the same per-row arithmetic; liboracle.so ignores the pragma */
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t u = r0; u < r1; ++u) {
    double *yu = y + (u - r0) * ldy;
    double *cu = cond ? cond + (u - r0) * ldy : NULL;
    for (int64_t k = 0; k < f; ++k) { yu[k] = 0.0; if (cu) cu[k] = 0.0; }
    for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
      double ae = a ? a[e] : 1.0;
      const float *xv = x + (int64_t)col[e] * ldx;
      for (int64_t k = 0; k < f; ++k) {
        double t = ae * (double)xv[k];
        yu[k] += t;
        if (cu) cu[k] += fabs(t);
      }
    }
  }
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * 3b. GSpMM with a selectable reduce operator (NEXT-2).
 *    P:640-646 [§4.1 Eq. formula:1: h_u = phi(psi(h_v, h_e)); "users could
 *    choose the reduce or compute operator"], P:648 ["min and max as reduce
 *    functions"], P:1355 Fig. gspmm ["mean and sum as reduce functions"];
 *    an empty row gives 0 for every reduce; mean divides
 *    by the number of entries in the row.
 *    reduce: 0 sum, 1 mean, 2 max, 3 min.  psi: a == NULL -> copy (h_v),
 *    else multiply (a_e * h_v), formed in fp64 (exact for fp32 operands).
 * ------------------------------------------------------------------------- */
int orc_gspmm(int64_t r0, int64_t r1, const int64_t *row_ptr, const int32_t *col, const double *a,
              const float *x, int64_t f, int64_t ldx, int reduce, double *y, int64_t ldy) {
  if (r0 < 0 || r1 < r0 || f < 0 || ldx < f || ldy < f || !row_ptr || !x || !y || reduce < 0 || reduce > 3)
    return ORC_ERR_ARG;
  for (int64_t u = r0; u < r1; ++u) {
    double *yu = y + (u - r0) * ldy;
    const int64_t b = row_ptr[u], e1 = row_ptr[u + 1];
    for (int64_t k = 0; k < f; ++k) {
      double acc = 0.0;
      for (int64_t e = b; e < e1; ++e) {
        const double v = (a ? a[e] : 1.0) * (double)x[(int64_t)col[e] * ldx + k];
        if (reduce <= 1) acc += v;
        else if (e == b) acc = v;
        else if (reduce == 2 && v > acc) acc = v;
        else if (reduce == 3 && v < acc) acc = v;
      }
      if (reduce == 1 && e1 > b) acc /= (double)(e1 - b);
      yu[k] = (e1 > b) ? acc : 0.0;
    }
  }
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * 3c. K-step graph propagation (NEXT-4): y = sum_{k=0..K} theta_k A^k x.
 *    P:297 [graph diffusion matrix A_bar = sum_i alpha_i A^i "to collect
 *    information of distant neighbors"], P:255 [APPNP: personalized-PageRank
 *    propagation], S:171-188 [diffusion_matrix, ppr_coeffs].  Computed the
 *    plain way: t_0 = x, t_k = A t_{k-1}, y = sum_k theta_k t_k (fp64).
 *    cond (nullable) = the same recursion on |A|, |x|, |theta| (error scale).
 *    Works on all n rows (the recursion needs every row).
 * ------------------------------------------------------------------------- */
int orc_propagate(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *a, const float *x,
                  int64_t f, int64_t ldx, int64_t K, const double *theta, double *y, double *cond, int64_t ldy) {
  if (n < 0 || f < 0 || ldx < f || ldy < f || K < 0 || !row_ptr || !x || !theta || !y) return ORC_ERR_ARG;
  const size_t sz = (size_t)(n > 0 ? n : 1) * (size_t)(f > 0 ? f : 1);
  double *t = (double *)malloc(sizeof(double) * sz), *t2 = (double *)malloc(sizeof(double) * sz);
  double *ta = (double *)malloc(sizeof(double) * sz), *ta2 = (double *)malloc(sizeof(double) * sz);
  if (!t || !t2 || !ta || !ta2) { free(t); free(t2); free(ta); free(ta2); return ORC_ERR_NOMEM; }
  for (int64_t u = 0; u < n; ++u)
    for (int64_t k = 0; k < f; ++k) {
      t[u * f + k] = (double)x[u * ldx + k];
      ta[u * f + k] = fabs((double)x[u * ldx + k]);
      y[u * ldy + k] = theta[0] * t[u * f + k];
      if (cond) cond[u * ldy + k] = fabs(theta[0]) * ta[u * f + k];
    }
  for (int64_t step = 1; step <= K; ++step) {
    for (int64_t u = 0; u < n; ++u)
      for (int64_t k = 0; k < f; ++k) {
        double s = 0.0, sa = 0.0;
        for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
          const double ae = a ? a[e] : 1.0;
          s += ae * t[(int64_t)col[e] * f + k];
          sa += fabs(ae) * ta[(int64_t)col[e] * f + k];
        }
        t2[u * f + k] = s;
        ta2[u * f + k] = sa;
      }
    double *sw = t; t = t2; t2 = sw;
    sw = ta; ta = ta2; ta2 = sw;
    for (int64_t u = 0; u < n; ++u)
      for (int64_t k = 0; k < f; ++k) {
        y[u * ldy + k] += theta[step] * t[u * f + k];
        if (cond) cond[u * ldy + k] += fabs(theta[step]) * ta[u * f + k];
      }
  }
  free(t); free(t2); free(ta); free(ta2);
  return ORC_OK;
}

/* PPR (APPNP) coefficients: theta_k = alpha (1 - alpha)^k, k = 0..K. */
int orc_ppr_coeffs(double alpha, int64_t K, double *theta) {
  if (!(alpha > 0.0 && alpha <= 1.0) || K < 0 || !theta) return ORC_ERR_ARG;
  double p = alpha;
  for (int64_t k = 0; k <= K; ++k) { theta[k] = p; p *= (1.0 - alpha); }
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * 4. Edge-wise softmax, per head.
 *    P:653-656 [§4.1: alpha'_uv = exp(alpha_uv) / sum_{w in N(u)} exp(alpha_uw);
 *    "first apply the scan to find the max value ... subtract this maximum ...
 *    apply the exponent function and reduce ... to acquire the sum"];
 *    A9 (denominator over the whole row), A10 (max is a reduction),
 *    A12 (empty rows emit nothing).  logits/alpha are [nnz][heads].
 * ------------------------------------------------------------------------- */
int orc_edge_softmax(int64_t r0, int64_t r1, const int64_t *row_ptr, int64_t heads,
                     const double *logits, double *alpha) {
  if (r0 < 0 || r1 < r0 || heads <= 0 || !row_ptr || !logits || !alpha) return ORC_ERR_ARG;
  for (int64_t u = r0; u < r1; ++u) {
    int64_t b = row_ptr[u], e1 = row_ptr[u + 1];
    if (b == e1) continue;
    for (int64_t h = 0; h < heads; ++h) {
      double mx = -INFINITY;
      for (int64_t e = b; e < e1; ++e) if (logits[e * heads + h] > mx) mx = logits[e * heads + h];
      double s = 0.0;
      for (int64_t e = b; e < e1; ++e) s += exp(logits[e * heads + h] - mx);
      for (int64_t e = b; e < e1; ++e) alpha[e * heads + h] = exp(logits[e * heads + h] - mx) / s;
    }
  }
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * 5. GAT per-edge attention score ("masked self-attentional layers";
 *    the formula is not printed in the paper -> A13 / S:503, S:544 split form):
 *    s[e,h] = LeakyReLU(el[u,h] + er[v,h]; slope), e = (u,v) in row u.
 *    el is [n_rows][heads] (aggregating row), er is [n_cols][heads] (neighbour).
 * ------------------------------------------------------------------------- */
int orc_gat_scores(int64_t r0, int64_t r1, const int64_t *row_ptr, const int32_t *col,
                   int64_t heads, const float *el, const float *er, double slope, double *s) {
  if (r0 < 0 || r1 < r0 || heads <= 0 || !row_ptr || !el || !er || !s) return ORC_ERR_ARG;
  for (int64_t u = r0; u < r1; ++u)
    for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e)
      for (int64_t h = 0; h < heads; ++h) {
        double t = (double)el[u * heads + h] + (double)er[(int64_t)col[e] * heads + h];
        s[e * heads + h] = t >= 0.0 ? t : slope * t;
      }
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * 6. Multi-head SpMM.  P:648-649 [§4.1 multi-head SpMM: heads share the
 *    sparsity pattern]; A14 (Z, Y are [n][H][D], alpha [nnz][H]).
 *    y[u,h,d] = sum_e alpha[e,h] * z[col_e,h,d]; cond likewise with |.|.
 * ------------------------------------------------------------------------- */
int orc_multihead_spmm(int64_t r0, int64_t r1, const int64_t *row_ptr, const int32_t *col,
                       int64_t heads, const double *alpha, const float *z, int64_t d,
                       int64_t ldz, double *y, double *cond, int64_t ldy) {
  if (r0 < 0 || r1 < r0 || heads <= 0 || d < 0 || ldz < heads * d || ldy < heads * d ||
      !row_ptr || !alpha || !z || !y)
    return ORC_ERR_ARG;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t u = r0; u < r1; ++u) {
    double *yu = y + (u - r0) * ldy;
    double *cu = cond ? cond + (u - r0) * ldy : NULL;
    for (int64_t k = 0; k < heads * d; ++k) { yu[k] = 0.0; if (cu) cu[k] = 0.0; }
    for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
      const float *zv = z + (int64_t)col[e] * ldz;
      for (int64_t h = 0; h < heads; ++h) {
        double ah = alpha[e * heads + h];
        for (int64_t k = 0; k < d; ++k) {
          double t = ah * (double)zv[h * d + k];
          yu[h * d + k] += t;
          if (cu) cu[h * d + k] += fabs(t);
        }
      }
    }
  }
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * 7. Attention projection (A13; S:503, S:544 split form of a^T [z_u || z_v]):
 *    el[u,h] = sum_d a_l[h,d] z[u,h,d];  er[u,h] = sum_d a_r[h,d] z[u,h,d].
 *    *_cond = sum_d |a z| (dot-product tolerance).  Rows [r0, r1).
 * ------------------------------------------------------------------------- */
int orc_attn_project(int64_t r0, int64_t r1, int64_t heads, int64_t d, const float *z, int64_t ldz,
                     const float *a_l, const float *a_r, double *el, double *er,
                     double *el_cond, double *er_cond) {
  if (r0 < 0 || r1 < r0 || heads <= 0 || d < 0 || ldz < heads * d || !z || !a_l || !a_r || !el || !er)
    return ORC_ERR_ARG;
  for (int64_t u = r0; u < r1; ++u)
    for (int64_t h = 0; h < heads; ++h) {
      double sl = 0.0, sr = 0.0, cl = 0.0, cr = 0.0;
      for (int64_t k = 0; k < d; ++k) {
        double zv = (double)z[u * ldz + h * d + k];
        double tl = (double)a_l[h * d + k] * zv, tr = (double)a_r[h * d + k] * zv;
        sl += tl; sr += tr; cl += fabs(tl); cr += fabs(tr);
      }
      int64_t o = (u - r0) * heads + h;
      el[o] = sl; er[o] = sr;
      if (el_cond) el_cond[o] = cl;
      if (er_cond) er_cond[o] = cr;
    }
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * 10. GAT backward (NEXT-3).  P:652 [§4.1: SDDMM T = A (.) (P Q^T) "is used
 *     for back-propagating the gradients to the sparse adjacency matrix since
 *     the adjacency matrix of the GAT model is computed by the attention
 *     mechanism"]; S:153-161 (sddmm), S:237-245 (spmm_var backward).
 *
 * 10a. Multi-head SDDMM: out[e,h] = sum_k p[u,h,k] q[v,h,k], e = (u,v).
 *      Structural: A's values are not multiplied in.
 * ------------------------------------------------------------------------- */
int orc_sddmm(int64_t n, const int64_t *row_ptr, const int32_t *col, int64_t heads, int64_t d, const float *p,
              int64_t ldp, const float *q, int64_t ldq, double *out) {
  if (n < 0 || heads <= 0 || d < 0 || ldp < heads * d || ldq < heads * d || !row_ptr || !p || !q || !out)
    return ORC_ERR_ARG;
  for (int64_t u = 0; u < n; ++u)
    for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e)
      for (int64_t h = 0; h < heads; ++h) {
        double s = 0.0;
        for (int64_t k = 0; k < d; ++k)
          s += (double)p[u * ldp + h * d + k] * (double)q[(int64_t)col[e] * ldq + h * d + k];
        out[e * heads + h] = s;
      }
  return ORC_OK;
}

/* 10b. Transpose of a CSR with n_cols columns: rows of A^T are A's columns,
 *      entries in increasing original row; perm[e'] = index in A of entry e'
 *      of A^T.  Plain counting by column. */
int orc_csr_transpose(int64_t n_rows, int64_t n_cols, const int64_t *row_ptr, const int32_t *col,
                      int64_t *rp_t, int32_t *col_t, int64_t *perm) {
  if (n_rows < 0 || n_cols < 0 || !row_ptr || !rp_t) return ORC_ERR_ARG;
  const int64_t nnz = row_ptr[n_rows];
  for (int64_t c = 0; c <= n_cols; ++c) rp_t[c] = 0;
  for (int64_t e = 0; e < nnz; ++e) rp_t[col[e] + 1] += 1;
  for (int64_t c = 0; c < n_cols; ++c) rp_t[c + 1] += rp_t[c];
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_cols > 0 ? n_cols : 1));
  if (!fill) return ORC_ERR_NOMEM;
  for (int64_t c = 0; c < n_cols; ++c) fill[c] = rp_t[c];
  for (int64_t u = 0; u < n_rows; ++u)
    for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
      const int64_t k = fill[col[e]]++;
      col_t[k] = (int32_t)u;
      perm[k] = e;
    }
  free(fill);
  return ORC_OK;
}

/* 10c. Edge-softmax backward (the Jacobian of §4 per row and head):
 *      ds[e] = alpha[e] * (dalpha[e] - sum_{e' in row} alpha[e'] dalpha[e']). */
int orc_edge_softmax_backward(int64_t n, const int64_t *row_ptr, int64_t heads, const double *alpha,
                              const double *dalpha, double *ds) {
  if (n < 0 || heads <= 0 || !row_ptr || !alpha || !dalpha || !ds) return ORC_ERR_ARG;
  for (int64_t u = 0; u < n; ++u)
    for (int64_t h = 0; h < heads; ++h) {
      double dot = 0.0;
      for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) dot += alpha[e * heads + h] * dalpha[e * heads + h];
      for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e)
        ds[e * heads + h] = alpha[e * heads + h] * (dalpha[e * heads + h] - dot);
    }
  return ORC_OK;
}

/* 10d. Backward of the fused GAT aggregate (§5 scores, §4 softmax, §6 SpMM)
 *      given dY [n][H][D]:
 *        dalpha[e,h] = sum_k dY[u,h,k] z[v,h,k]                (SDDMM)
 *        dz[v,h,:]  += alpha[e,h] dY[u,h,:]                     (A^T SpMM)
 *        ds = softmax backward;  dt = ds * (t >= 0 ? 1 : slope),  t = el[u]+er[v]
 *        d_el[u,h] = sum_{e in row u} dt[e,h];  d_er[v,h] = sum_{e=(u,v)} dt[e,h]
 *      alpha is recomputed here from el, er (fp64).  dt (nullable) [nnz][H]. */
int orc_gat_backward(int64_t n, const int64_t *row_ptr, const int32_t *col, int64_t heads, const float *el,
                     const float *er, double slope, const float *z, int64_t d, int64_t ldz, const float *dy,
                     int64_t lddy, double *dz, double *d_el, double *d_er, double *dt_out) {
  if (n < 0 || heads <= 0 || d < 0 || !row_ptr || !el || !er || !z || !dy || !dz || !d_el || !d_er)
    return ORC_ERR_ARG;
  const int64_t nnz = row_ptr[n], H = heads;
  double *s = (double *)malloc(sizeof(double) * (size_t)(nnz * H > 0 ? nnz * H : 1));
  double *al = (double *)malloc(sizeof(double) * (size_t)(nnz * H > 0 ? nnz * H : 1));
  double *da = (double *)malloc(sizeof(double) * (size_t)(nnz * H > 0 ? nnz * H : 1));
  double *ds = (double *)malloc(sizeof(double) * (size_t)(nnz * H > 0 ? nnz * H : 1));
  if (!s || !al || !da || !ds) { free(s); free(al); free(da); free(ds); return ORC_ERR_NOMEM; }
  int rc = orc_gat_scores(0, n, row_ptr, col, H, el, er, slope, s);
  if (!rc) rc = orc_edge_softmax(0, n, row_ptr, H, s, al);
  if (!rc) rc = orc_sddmm(n, row_ptr, col, H, d, dy, lddy, z, ldz, da);
  if (!rc) rc = orc_edge_softmax_backward(n, row_ptr, H, al, da, ds);
  if (!rc) {
    for (int64_t v = 0; v < n; ++v)
      for (int64_t k = 0; k < H * d; ++k) dz[v * H * d + k] = 0.0;
    for (int64_t v = 0; v < n * H; ++v) { d_el[v] = 0.0; d_er[v] = 0.0; }
    for (int64_t u = 0; u < n; ++u)
      for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
        const int64_t v = col[e];
        for (int64_t h = 0; h < H; ++h) {
          const double t = (double)el[u * H + h] + (double)er[v * H + h];
          const double dt = ds[e * H + h] * (t >= 0.0 ? 1.0 : slope);
          if (dt_out) dt_out[e * H + h] = dt;
          d_el[u * H + h] += dt;
          d_er[v * H + h] += dt;
          for (int64_t k = 0; k < d; ++k) dz[v * H * d + h * d + k] += al[e * H + h] * (double)dy[u * lddy + h * d + k];
        }
      }
  }
  free(s); free(al); free(da); free(ds);
  return rc;
}

/* 10e. Backward of the attention projection (§7): el = z.a_l, er = z.a_r per
 *      head, so dz[u,h,:] = d_el[u,h] a_l[h,:] + d_er[u,h] a_r[h,:] and
 *      d_al[h,:] = sum_u d_el[u,h] z[u,h,:] (d_ar likewise). */
int orc_attn_project_backward(int64_t n, int64_t heads, int64_t d, const float *z, int64_t ldz, const float *a_l,
                              const float *a_r, const double *d_el, const double *d_er, double *dz, double *d_al,
                              double *d_ar) {
  if (n < 0 || heads <= 0 || d < 0 || ldz < heads * d || !z || !a_l || !a_r || !d_el || !d_er || !dz || !d_al || !d_ar)
    return ORC_ERR_ARG;
  for (int64_t k = 0; k < heads * d; ++k) { d_al[k] = 0.0; d_ar[k] = 0.0; }
  for (int64_t u = 0; u < n; ++u)
    for (int64_t h = 0; h < heads; ++h)
      for (int64_t k = 0; k < d; ++k) {
        const int64_t c = h * d + k;
        dz[u * heads * d + c] = d_el[u * heads + h] * (double)a_l[c] + d_er[u * heads + h] * (double)a_r[c];
        d_al[c] += d_el[u * heads + h] * (double)z[u * ldz + c];
        d_ar[c] += d_er[u * heads + h] * (double)z[u * ldz + c];
      }
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * 11. Layers for 2-layer inference (NEXT-1).  P:239-246 [Eq. gcn_layer:
 *     H^(l+1) = sigma(A^ H^(l) W^(l))]; P:253 (GAT); P:661-663 [Table
 *     spmm_time: 2-layer GCN / GAT inference, hidden 128, GAT 4 heads].
 *     act: 0 none, 1 ReLU (GCN hidden layers), 2 ELU alpha=1 (GAT hidden).
 * 11a. y = x W (+ bias) on rows [r0, r1); W row-major [f_in][f_out].
 * ------------------------------------------------------------------------- */
static double orc_act(double v, int act) {
  if (act == 1) return v > 0.0 ? v : 0.0;
  if (act == 2) return v > 0.0 ? v : expm1(v);
  return v;
}

int orc_linear(int64_t r0, int64_t r1, const float *x, int64_t ldx, int64_t f_in, const float *w, int64_t f_out,
               const float *bias, double *y, double *cond, int64_t ldy) {
  if (r0 < 0 || r1 < r0 || f_in < 0 || f_out < 0 || ldx < f_in || ldy < f_out || !x || !w || !y) return ORC_ERR_ARG;
  for (int64_t u = r0; u < r1; ++u)
    for (int64_t j = 0; j < f_out; ++j) {
      double s = bias ? (double)bias[j] : 0.0, c = bias ? fabs((double)bias[j]) : 0.0;
      for (int64_t k = 0; k < f_in; ++k) {
        const double t = (double)x[u * ldx + k] * (double)w[k * f_out + j];
        s += t;
        c += fabs(t);
      }
      y[(u - r0) * ldy + j] = s;
      if (cond) cond[(u - r0) * ldy + j] = c;
    }
  return ORC_OK;
}

/* 11b. GCN layer on rows [r0, r1): y[u] = act(sum_e a_e (x[col_e] W) + bias),
 *      the product computed per neighbour (Eq. gcn_layer written out).
 *      cond[u] = sum_e |a_e| (|x[col_e]| |W|) + |bias| (error scale, before act). */
int orc_gcn_layer(int64_t r0, int64_t r1, const int64_t *row_ptr, const int32_t *col, const double *a,
                  const float *x, int64_t ldx, int64_t f_in, const float *w, int64_t f_out, const float *bias, int act,
                  double *y, double *cond, int64_t ldy) {
  if (r0 < 0 || r1 < r0 || f_in < 0 || f_out < 0 || ldx < f_in || ldy < f_out || !row_ptr || !x || !w || !y)
    return ORC_ERR_ARG;
  double *t = (double *)malloc(sizeof(double) * (size_t)(f_out > 0 ? f_out : 1));
  double *tc = (double *)malloc(sizeof(double) * (size_t)(f_out > 0 ? f_out : 1));
  if (!t || !tc) { free(t); free(tc); return ORC_ERR_NOMEM; }
  for (int64_t u = r0; u < r1; ++u) {
    double *yu = y + (u - r0) * ldy;
    double *cu = cond ? cond + (u - r0) * ldy : NULL;
    for (int64_t j = 0; j < f_out; ++j) {
      yu[j] = bias ? (double)bias[j] : 0.0;
      if (cu) cu[j] = bias ? fabs((double)bias[j]) : 0.0;
    }
    for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
      const double ae = a ? a[e] : 1.0;
      orc_linear(col[e], col[e] + 1, x, ldx, f_in, w, f_out, NULL, t, tc, f_out);
      for (int64_t j = 0; j < f_out; ++j) {
        yu[j] += ae * t[j];
        if (cu) cu[j] += fabs(ae) * tc[j];
      }
    }
    for (int64_t j = 0; j < f_out; ++j) yu[j] = orc_act(yu[j], act);
  }
  free(t); free(tc);
  return ORC_OK;
}

/* 11c. Elementwise act(x + bias) (for composing layers in tests). */
int orc_bias_act(int64_t n, int64_t f, double *y, int64_t ldy, const float *bias, int act) {
  if (n < 0 || f < 0 || ldy < f || !y) return ORC_ERR_ARG;
  for (int64_t u = 0; u < n; ++u)
    for (int64_t j = 0; j < f; ++j) y[u * ldy + j] = orc_act(y[u * ldy + j] + (bias ? (double)bias[j] : 0.0), act);
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * 8. Row partition balanced by nnz (DESIGN.md multi-GPU):
 *    bound_p = lower_bound(row_ptr[0..n], ceil(p * nnz / P)) for 0 < p < P,
 *    bound_0 = 0, bound_P = n.  lower_bound = first r with row_ptr[r] >= t.
 *    Plain linear scan.
 * ------------------------------------------------------------------------- */
int orc_partition_rows(int64_t n, const int64_t *row_ptr, int64_t parts, int64_t *bounds) {
  if (n < 0 || parts <= 0 || !row_ptr || !bounds) return ORC_ERR_ARG;
  int64_t nnz = row_ptr[n];
  bounds[0] = 0;
  for (int64_t p = 1; p < parts; ++p) {
    int64_t t = (p * nnz + parts - 1) / parts;
    int64_t r = 0;
    while (r < n && row_ptr[r] < t) ++r;
    bounds[p] = r;
  }
  bounds[parts] = n;
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * 9. CSR slice for rank `rank` with columns remapped into the padded
 *    all-gather layout: rows [b_rank, b_rank+1); a column c
 *    owned by rank q (b_q <= c < b_q+1) becomes q * rows_padded + (c - b_q).
 *    row_ptr_out [rows+1] starts at 0; values are copied unchanged.
 * ------------------------------------------------------------------------- */
int orc_csr_slice(int64_t n, const int64_t *row_ptr, const int32_t *col, const float *val,
                  const int64_t *bounds, int64_t parts, int64_t rank, int64_t rows_padded,
                  int64_t *row_ptr_out, int32_t *col_out, float *val_out) {
  if (n < 0 || parts <= 0 || rank < 0 || rank >= parts || !row_ptr || !bounds || !row_ptr_out)
    return ORC_ERR_ARG;
  int64_t r0 = bounds[rank], r1 = bounds[rank + 1];
  int64_t base = row_ptr[r0];
  for (int64_t u = r0; u <= r1; ++u) row_ptr_out[u - r0] = row_ptr[u] - base;
  for (int64_t e = row_ptr[r0]; e < row_ptr[r1]; ++e) {
    int64_t c = col[e];
    int64_t q = 0;
    while (!(bounds[q] <= c && c < bounds[q + 1])) ++q;
    if (col_out) col_out[e - base] = (int32_t)(q * rows_padded + (c - bounds[q]));
    if (val_out && val) val_out[e - base] = val[e];
  }
  return ORC_OK;
}
