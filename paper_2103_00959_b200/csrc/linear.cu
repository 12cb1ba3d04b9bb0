// linear.cu -- NEXT-1: the dense step of a GNN layer, Y = X W (Eq. gcn_layer,
// P:242 H W), and the GCN layer act(A^ (X W) + b).  With a workspace, X W runs
// on the tcgen05 tensor cores (linear_tc.cu: 3xTF32, fp32-accurate); without
// one (or for f_out > 256 / unaligned X) it is delegated to cuBLAS (fp32
// compute, CUBLAS_COMPUTE_32F).  The sparse aggregation, bias and activation
// run in the SpMM engine (fused epilogue).
#include <cublas_v2.h>

#include <algorithm>

#include "spmm_engine.cuh"

namespace gsp {

// one cuBLAS handle per (thread, device), created on first use
static cublasHandle_t blas_handle() {
  static thread_local cublasHandle_t h[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!h[dev] && cublasCreate(&h[dev]) != CUBLAS_STATUS_SUCCESS) h[dev] = nullptr;
  return h[dev];
}

size_t linear_tc_ws_bytes(int64_t f_in, int64_t f_out);
bool linear_tc_eligible(int64_t n, int64_t f_in, const float *x, int64_t ldx, int64_t f_out, void *ws,
                        size_t ws_bytes);
gsp_status linear_tc(int64_t n, int64_t f_in, const float *x, int64_t ldx, const float *w, int64_t ldw,
                     int64_t f_out, float *y, int64_t ldy, void *ws, cudaStream_t s);

}  // namespace gsp

using namespace gsp;

extern "C" gsp_status gsp_linear_workspace(int64_t f_in, int64_t f_out, size_t *ws_bytes) {
  clear_detail();
  if (f_in < 0 || f_out < 0 || !ws_bytes) return fail(GSP_ERR_INVALID_ARG, "gsp_linear_workspace: bad argument");
  *ws_bytes = linear_tc_ws_bytes(f_in, f_out);
  return GSP_OK;
}

extern "C" gsp_status gsp_linear(int64_t n, int64_t f_in, const float *x, int64_t ldx, const float *w, int64_t ldw,
                                 int64_t f_out, float *y, int64_t ldy, void *ws, size_t ws_bytes, gsp_stream stream) {
  const char *fn = "gsp_linear";
  clear_detail();
  if (n < 0 || f_in < 0 || f_out < 0 || ldx < f_in || ldw < f_out || ldy < f_out)
    return fail(GSP_ERR_INVALID_ARG, "%s: bad sizes", fn);
  if (n == 0 || f_out == 0) return GSP_OK;
  if (!x || !w || !y) return fail(GSP_ERR_INVALID_ARG, "%s: null pointer", fn);
  if (n >= (int64_t(1) << 31) || f_in >= (int64_t(1) << 31)) return fail(GSP_ERR_UNSUPPORTED, "%s: too large", fn);
  if (overlaps(x, (size_t)((n - 1) * ldx + f_in) * 4, y, (size_t)((n - 1) * ldy + f_out) * 4))
    return fail(GSP_ERR_ALIAS, "%s: x and y overlap", fn);
  if (linear_tc_eligible(n, f_in, x, ldx, f_out, ws, ws_bytes))
    return linear_tc(n, f_in, x, ldx, w, ldw, f_out, y, ldy, ws, cs(stream));
  cublasHandle_t h = blas_handle();
  if (!h) return fail(GSP_ERR_CUDA, "%s: cublasCreate failed", fn);
  if (cublasSetStream(h, cs(stream)) != CUBLAS_STATUS_SUCCESS) return fail(GSP_ERR_CUDA, "%s: cublasSetStream", fn);
  const float one = 1.0f, zero = 0.0f;
  // row-major Y[n x f_out] = X[n x f_in] W[f_in x f_out]  <=>  column-major Y^T = W^T X^T
  const cublasStatus_t r = cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)f_out, (int)n, (int)f_in, &one, w,
                                        CUDA_R_32F, (int)ldw, x, CUDA_R_32F, (int)ldx, &zero, y, CUDA_R_32F, (int)ldy,
                                        CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
  if (r != CUBLAS_STATUS_SUCCESS) return fail(GSP_ERR_CUDA, "%s: cublasGemmEx status %d", fn, (int)r);
  return GSP_OK;
}

extern "C" gsp_status gsp_gcn_layer_workspace(int64_t n, int64_t f_in, int64_t f_out, size_t *ws_bytes) {
  clear_detail();
  if (n < 0 || f_in < 0 || f_out < 0 || !ws_bytes)
    return fail(GSP_ERR_INVALID_ARG, "gsp_gcn_layer_workspace: bad argument");
  // H = X W [n][round_up(f_out, 4)] (256-aligned), then the GEMM's split-W workspace
  *ws_bytes = (size_t)n * ((f_out + 3) / 4 * 4) * 4 + 256 + linear_tc_ws_bytes(f_in, f_out);
  return GSP_OK;
}

extern "C" gsp_status gsp_gcn_layer(const gsp_csr *a, const float *x, int64_t f_in, int64_t ldx, const float *w,
                                    int64_t f_out, const float *bias, gsp_act act, float *y, int64_t ldy, void *ws,
                                    size_t ws_bytes, gsp_stream stream) {
  const char *fn = "gsp_gcn_layer";
  clear_detail();
  gsp_status st = check_csr(a, false, fn);
  if (st) return st;
  // every argument is checked before the first enqueue (gsp.h: nothing is
  // touched on a host-detected error)
  if (act < GSP_ACT_NONE || act > GSP_ACT_ELU) return fail(GSP_ERR_INVALID_ARG, "%s: bad activation", fn);
  if (f_in < 0 || f_out < 0 || ldx < f_in || ldy < f_out) return fail(GSP_ERR_INVALID_ARG, "%s: bad sizes", fn);
  if (a->n_rows == 0 || f_out == 0) return GSP_OK;
  if (!y || !w || (a->n_cols > 0 && !x)) return fail(GSP_ERR_INVALID_ARG, "%s: null pointer", fn);
  if (a->n_cols >= (int64_t(1) << 31) || f_in >= (int64_t(1) << 31)) return fail(GSP_ERR_UNSUPPORTED, "%s: too large", fn);
  size_t need = 0;
  gsp_gcn_layer_workspace(a->n_cols, f_in, f_out, &need);
  if (!ws || ws_bytes < need) return fail(GSP_ERR_WORKSPACE, "%s: workspace needs %zu bytes", fn, need);
  const size_t yb = (size_t)((a->n_rows - 1) * ldy + f_out) * 4;
  if (overlaps(y, yb, ws, ws_bytes)) return fail(GSP_ERR_ALIAS, "%s: y overlaps the workspace", fn);
  if (a->n_cols > 0 && (overlaps(x, (size_t)((a->n_cols - 1) * ldx + f_in) * 4, ws, ws_bytes)))
    return fail(GSP_ERR_ALIAS, "%s: x overlaps the workspace", fn);
  float *h = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  const int64_t ldh = (f_out + 3) / 4 * 4;
  const size_t hb = (size_t)a->n_cols * ldh * 4;
  uint8_t *lws = reinterpret_cast<uint8_t *>(h) + hb;
  const size_t lws_bytes = ws_bytes - (size_t)(lws - reinterpret_cast<uint8_t *>(ws));
  if (ldh > f_out && a->n_cols > 0 &&  // keep the padding columns defined (the SpMM may read them, gsp.h)
      cudaMemset2DAsync(h + f_out, (size_t)ldh * 4, 0, (size_t)(ldh - f_out) * 4, (size_t)a->n_cols, cs(stream)) !=
          cudaSuccess)
    return check_launch("cudaMemset2DAsync(gcn_layer padding)");
  if ((st = gsp_linear(a->n_cols, f_in, x, ldx, w, f_out, f_out, h, ldh, lws, lws_bytes, stream))) return st;
  return gsp_spmm_bias_act(a, h, f_out, ldh, bias, act, y, ldy, stream);
}
