// partition.cu -- multi-GPU row partition and CSR slicing (DESIGN.md
// §Multi-GPU): contiguous row blocks balanced by nnz, and
// the per-rank slice with columns remapped into the padded all-gather layout.
#include <algorithm>

#include "common.cuh"

namespace gsp {

constexpr int kMaxParts = 128;

struct Bounds {
  int64_t b[kMaxParts + 1];
};

__global__ void partition_kernel(const int64_t *__restrict__ rp, int64_t n, int64_t nnz, int parts,
                                 int64_t *__restrict__ out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > parts) return;
  if (p == 0) { out[0] = 0; return; }
  if (p == parts) { out[parts] = n; return; }
  const int64_t t = (p * nnz + parts - 1) / parts;  // ceil(p * nnz / parts)
  int64_t lo = 0, hi = n;                             // first r in [0, n) with rp[r] >= t, else n
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (rp[mid] >= t) hi = mid; else lo = mid + 1;
  }
  out[p] = lo;
}

__global__ void slice_rowptr_kernel(const int64_t *__restrict__ rp, int64_t r0, int64_t rows,
                                    int64_t *__restrict__ out) {
  const int64_t base = rp[r0];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= rows; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = rp[r0 + i] - base;
}

__global__ void slice_cols_kernel(const int64_t *__restrict__ rp, int64_t r0, int64_t r1,
                                  const int32_t *__restrict__ col, const float *__restrict__ val, const Bounds B,
                                  int parts, int64_t rows_padded, int32_t *__restrict__ col_out,
                                  float *__restrict__ val_out) {
  const int64_t base = rp[r0], k = rp[r1] - base;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < k; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = col[base + e];
    int lo = 0, hi = parts - 1;  // owner q: first q with B.b[q+1] > c
    while (lo < hi) {
      const int mid = (lo + hi) / 2;
      if (B.b[mid + 1] > c) hi = mid; else lo = mid + 1;
    }
    col_out[e] = (int32_t)((int64_t)lo * rows_padded + (c - B.b[lo]));
    if (val_out) val_out[e] = val[base + e];
  }
}

}  // namespace gsp

using namespace gsp;

extern "C" gsp_status gsp_partition_rows(const gsp_csr *a, int32_t parts, int64_t *row_bounds_dev,
                                         int64_t *row_bounds_host, gsp_stream stream) {
  const char *fn = "gsp_partition_rows";
  clear_detail();
  gsp_status st = check_csr(a, false, fn);
  if (st) return st;
  if (parts <= 0 || parts > kMaxParts) return fail(GSP_ERR_INVALID_ARG, "%s: parts must be in [1, %d]", fn, kMaxParts);
  if (!row_bounds_dev) return fail(GSP_ERR_INVALID_ARG, "%s: row_bounds_dev is NULL", fn);
  cudaStream_t s = cs(stream);
  partition_kernel<<<1, 256, 0, s>>>(a->row_ptr, a->n_rows, a->nnz, parts, row_bounds_dev);
  if ((st = check_launch("partition"))) return st;
  if (row_bounds_host &&
      (cudaMemcpyAsync(row_bounds_host, row_bounds_dev, (parts + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s) !=
           cudaSuccess ||
       cudaStreamSynchronize(s) != cudaSuccess))
    return check_launch("partition copy");
  return GSP_OK;
}

extern "C" gsp_status gsp_csr_slice(const gsp_csr *a, const int64_t *row_bounds, int32_t parts, int32_t rank,
                                    int64_t rows_padded, int64_t *row_ptr_out, int32_t *col_out, float *val_out,
                                    gsp_stream stream) {
  const char *fn = "gsp_csr_slice";
  clear_detail();
  gsp_status st = check_csr(a, false, fn);
  if (st) return st;
  if (parts <= 0 || parts > kMaxParts || rank < 0 || rank >= parts || !row_bounds)
    return fail(GSP_ERR_INVALID_ARG, "%s: bad parts / rank / row_bounds", fn);
  Bounds B;
  int64_t maxpart = 0;
  for (int p = 0; p <= parts; ++p) {
    B.b[p] = row_bounds[p];
    if (p && B.b[p] < B.b[p - 1]) return fail(GSP_ERR_INVALID_ARG, "%s: row_bounds not nondecreasing", fn);
    if (p) maxpart = std::max(maxpart, B.b[p] - B.b[p - 1]);
  }
  if (B.b[0] != 0 || B.b[parts] != a->n_rows) return fail(GSP_ERR_INVALID_ARG, "%s: bounds must span [0, n)", fn);
  if (a->n_rows != a->n_cols) return fail(GSP_ERR_INVALID_ARG, "%s: matrix must be square", fn);
  if (rows_padded < maxpart) return fail(GSP_ERR_INVALID_ARG, "%s: rows_padded < largest part", fn);
  if ((int64_t)parts * rows_padded >= (int64_t(1) << 31)) return fail(GSP_ERR_UNSUPPORTED, "%s: P*rows_padded >= 2^31", fn);
  if (!row_ptr_out) return fail(GSP_ERR_INVALID_ARG, "%s: row_ptr_out is NULL", fn);
  const int64_t r0 = B.b[rank], r1 = B.b[rank + 1], rows = r1 - r0;
  cudaStream_t s = cs(stream);
  slice_rowptr_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows + 1, 256), 8192)), 256, 0, s>>>(
      a->row_ptr, r0, rows, row_ptr_out);
  if ((st = check_launch("slice_rowptr"))) return st;
  if (a->nnz > 0) {
    if (!col_out) return fail(GSP_ERR_INVALID_ARG, "%s: col_out is NULL", fn);
    slice_cols_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(a->nnz / parts + 1, 256), 65535)),
                        256, 0, s>>>(a->row_ptr, r0, r1, a->col_idx, a->val ? a->val : nullptr, B, parts, rows_padded,
                                     col_out, a->val ? val_out : nullptr);
    if ((st = check_launch("slice_cols"))) return st;
  }
  return GSP_OK;
}
