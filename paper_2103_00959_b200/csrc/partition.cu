// partition.cu -- multi-GPU row partition and CSR slicing (DESIGN.md
// §Multi-GPU): contiguous row blocks balanced by nnz, and
// the per-rank slice with columns remapped into the padded all-gather layout.
#include <algorithm>
#include <vector>

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

// ---------------------------------------------------------- column blocks
// A = sum_k A_k, A_k = the entries of A with column in [bounds[k], bounds[k+1]).
// Columns are sorted within a row, so a row's block-k entries are one
// contiguous run; a warp per row counts them (ballots over the row's columns)
// and later copies them, keeping their order.
constexpr int kMaxColBlocks = 8;
struct ColBounds {
  int64_t b[kMaxColBlocks + 1];
};

// offsets of the row's block boundaries: lane-strided count of columns < b_k
__device__ __forceinline__ void colblock_offsets(const int32_t *__restrict__ col, int64_t start, int64_t d,
                                                 const ColBounds &B, int K, int lane, int64_t (&off)[kMaxColBlocks + 1]) {
  off[0] = 0;
  off[K] = d;
  for (int k = 1; k < K; ++k) {
    int64_t c = 0;
    for (int64_t j = lane; j < d; j += 32) c += (int64_t)(__ldg(col + start + j) < B.b[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    off[k] = c;
  }
}

__global__ void __launch_bounds__(256) colblock_count_kernel(const int64_t *__restrict__ rp,
                                                             const int32_t *__restrict__ col, int64_t n_rows,
                                                             const ColBounds B, int K, uint32_t *__restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_rows; r += nw) {
    const int64_t start = __ldg(rp + r), d = __ldg(rp + r + 1) - start;
    int64_t off[kMaxColBlocks + 1];
    colblock_offsets(col, start, d, B, K, lane, off);
    if (lane < K) {
      int64_t c = 0;
      for (int k = 0; k < K; ++k)
        if (k == lane) c = off[k + 1] - off[k];
      counts[(int64_t)lane * (n_rows + 1) + r] = (uint32_t)c;
    }
  }
}

// widen a block's scanned counts (uint32, [n_rows + 1]) into its int64 row_ptr
__global__ void colblock_rowptr_kernel(const uint32_t *__restrict__ scanned, int64_t count,
                                       int64_t *__restrict__ row_ptr) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    row_ptr[i] = (int64_t)scanned[i];
}

struct ColBlockOut {
  int64_t *row_ptr[kMaxColBlocks];
  int32_t *col[kMaxColBlocks];
  float *val[kMaxColBlocks];
};

__global__ void __launch_bounds__(256) colblock_scatter_kernel(const int64_t *__restrict__ rp,
                                                               const int32_t *__restrict__ col,
                                                               const float *__restrict__ val, int64_t n_rows,
                                                               const ColBounds B, int K, const ColBlockOut O) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_rows; r += nw) {
    const int64_t start = __ldg(rp + r), d = __ldg(rp + r + 1) - start;
    int64_t off[kMaxColBlocks + 1];
    colblock_offsets(col, start, d, B, K, lane, off);
    for (int k = 0; k < K; ++k) {
      const int64_t dst = O.row_ptr[k][r];
      for (int64_t j = off[k] + lane; j < off[k + 1]; j += 32) {
        O.col[k][dst + j - off[k]] = __ldg(col + start + j);
        if (val) O.val[k][dst + j - off[k]] = __ldg(val + start + j);
      }
    }
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

// ---- column blocks (host) ---------------------------------------------------
namespace {
size_t a256(size_t b) { return (b + 255) & ~size_t(255); }
struct ColBlockLayout {
  size_t row_ptr, col, val, counts, scan, total;
};
ColBlockLayout colblock_layout(int64_t n_rows, int64_t nnz, int K) {
  ColBlockLayout L{};
  size_t o = 0;
  L.row_ptr = o;
  o += (size_t)K * a256((size_t)(n_rows + 1) * 8);
  L.col = o;
  o += a256((size_t)std::max<int64_t>(nnz, 1) * 4 + (size_t)K * 16);
  L.val = o;
  o += a256((size_t)std::max<int64_t>(nnz, 1) * 4 + (size_t)K * 16);
  L.counts = o;
  o += a256((size_t)K * (n_rows + 1) * 4);
  L.scan = o;
  o += a256(scan_ws_bytes(n_rows + 1));
  L.total = o + 256;
  return L;
}
}  // namespace

extern "C" gsp_status gsp_csr_colblock_workspace(const gsp_csr *a, int32_t blocks, size_t *ws_bytes) {
  clear_detail();
  if (!a || !ws_bytes || blocks < 1 || blocks > kMaxColBlocks)
    return fail(GSP_ERR_INVALID_ARG, "gsp_csr_colblock_workspace: bad argument (blocks in [1, %d])", kMaxColBlocks);
  *ws_bytes = colblock_layout(a->n_rows, a->nnz, blocks).total;
  return GSP_OK;
}

extern "C" gsp_status gsp_csr_colblock(const gsp_csr *a, const int64_t *col_bounds, int32_t blocks, void *ws,
                                       size_t ws_bytes, gsp_csr *out, gsp_stream stream) {
  const char *fn = "gsp_csr_colblock";
  clear_detail();
  gsp_status st = check_csr(a, false, fn);
  if (st) return st;
  if (blocks < 1 || blocks > kMaxColBlocks || !col_bounds || !out)
    return fail(GSP_ERR_INVALID_ARG, "%s: blocks in [1, %d], col_bounds and out required", fn, kMaxColBlocks);
  ColBounds B;
  for (int k = 0; k <= blocks; ++k) {
    B.b[k] = col_bounds[k];
    if (k && B.b[k] < B.b[k - 1]) return fail(GSP_ERR_INVALID_ARG, "%s: col_bounds not nondecreasing", fn);
  }
  if (B.b[0] != 0 || B.b[blocks] != a->n_cols) return fail(GSP_ERR_INVALID_ARG, "%s: col_bounds must span [0, n_cols)", fn);
  const ColBlockLayout L = colblock_layout(a->n_rows, a->nnz, blocks);
  if (!ws || ws_bytes < L.total) return fail(GSP_ERR_WORKSPACE, "%s: workspace needs %zu bytes", fn, L.total);
  cudaStream_t s = cs(stream);
  uint8_t *W = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  uint32_t *counts = reinterpret_cast<uint32_t *>(W + L.counts);
  const int64_t n = a->n_rows;
  if (cudaMemsetAsync(counts, 0, (size_t)blocks * (n + 1) * 4, s) != cudaSuccess) return check_launch("memset");
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 8), 8 * (int64_t)sm_count() * 8));
  if (n > 0) {
    colblock_count_kernel<<<grid, 256, 0, s>>>(a->row_ptr, a->col_idx, n, B, blocks, counts);
    if ((st = check_launch("colblock_count"))) return st;
  }
  for (int k = 0; k < blocks; ++k)  // counts[k][n] == 0: the scan's last entry is block k's nnz
    if ((st = scan_exclusive(counts + (size_t)k * (n + 1), counts + (size_t)k * (n + 1), n + 1, W + L.scan, s)))
      return st;
  std::vector<uint32_t> tot(blocks);
  for (int k = 0; k < blocks; ++k)
    if (cudaMemcpyAsync(&tot[k], counts + (size_t)k * (n + 1) + n, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess)
      return check_launch("colblock totals");
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_launch("colblock sync");
  ColBlockOut O{};
  int64_t base = 0;
  for (int k = 0; k < blocks; ++k) {
    O.row_ptr[k] = reinterpret_cast<int64_t *>(W + L.row_ptr + (size_t)k * a256((size_t)(n + 1) * 8));
    const int64_t c0 = (base + 3) & ~int64_t(3);  // 16-byte aligned runs (TMA staging of the window)
    O.col[k] = reinterpret_cast<int32_t *>(W + L.col) + c0;
    O.val[k] = a->val ? reinterpret_cast<float *>(W + L.val) + c0 : nullptr;
    base = c0 + tot[k];
  }
  for (int k = 0; k < blocks; ++k) {
    colblock_rowptr_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n + 1, 256), 4096)), 256, 0,
                             s>>>(counts + (size_t)k * (n + 1), n + 1, O.row_ptr[k]);
    if ((st = check_launch("colblock_rowptr"))) return st;
  }
  if (n > 0 && a->nnz > 0) {
    colblock_scatter_kernel<<<grid, 256, 0, s>>>(a->row_ptr, a->col_idx, a->val, n, B, blocks, O);
    if ((st = check_launch("colblock_scatter"))) return st;
  }
  for (int k = 0; k < blocks; ++k) {
    out[k].n_rows = n;
    out[k].n_cols = a->n_cols;
    out[k].nnz = tot[k];
    out[k].row_ptr = O.row_ptr[k];
    out[k].col_idx = O.col[k];
    out[k].val = O.val[k];
  }
  return GSP_OK;
}
