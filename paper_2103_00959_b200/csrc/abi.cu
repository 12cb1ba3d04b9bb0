// abi.cu -- status strings, thread-local error detail, shared host checks.
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace gsp {

static thread_local char g_detail[512] = "";

void set_detail(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_detail, sizeof(g_detail), fmt, ap);
  va_end(ap);
}

void clear_detail() { g_detail[0] = 0; }

gsp_status fail(gsp_status st, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_detail, sizeof(g_detail), fmt, ap);
  va_end(ap);
  return st;
}

gsp_status check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(GSP_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return GSP_OK;
}

int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev] = v;
  }
  return cache[dev];
}

gsp_status check_csr(const gsp_csr *a, bool need_val, const char *fn) {
  if (!a) return fail(GSP_ERR_INVALID_ARG, "%s: csr view is NULL", fn);
  if (a->n_rows < 0 || a->n_cols < 0 || a->nnz < 0)
    return fail(GSP_ERR_INVALID_ARG, "%s: negative csr size", fn);
  if (a->n_rows >= (int64_t(1) << 31) || a->n_cols >= (int64_t(1) << 31))
    return fail(GSP_ERR_UNSUPPORTED, "%s: n_rows / n_cols must be < 2^31", fn);
  if (!a->row_ptr) return fail(GSP_ERR_INVALID_ARG, "%s: row_ptr is NULL", fn);
  if (a->nnz > 0 && !a->col_idx) return fail(GSP_ERR_INVALID_ARG, "%s: col_idx is NULL", fn);
  if (need_val && a->nnz > 0 && !a->val) return fail(GSP_ERR_INVALID_ARG, "%s: val is NULL", fn);
  return GSP_OK;
}

}  // namespace gsp

extern "C" {

const char *gsp_status_string(gsp_status st) {
  switch (st) {
    case GSP_OK: return "GSP_OK";
    case GSP_ERR_INVALID_ARG: return "GSP_ERR_INVALID_ARG";
    case GSP_ERR_INDEX_RANGE: return "GSP_ERR_INDEX_RANGE";
    case GSP_ERR_NEGATIVE_WEIGHT: return "GSP_ERR_NEGATIVE_WEIGHT";
    case GSP_ERR_NONFINITE: return "GSP_ERR_NONFINITE";
    case GSP_ERR_ALIAS: return "GSP_ERR_ALIAS";
    case GSP_ERR_WORKSPACE: return "GSP_ERR_WORKSPACE";
    case GSP_ERR_UNSUPPORTED: return "GSP_ERR_UNSUPPORTED";
    case GSP_ERR_CUDA: return "GSP_ERR_CUDA";
  }
  return "GSP_ERR_UNKNOWN";
}

const char *gsp_last_error_detail(void) { return gsp::g_detail; }

int gsp_version(void) { return GSP_VERSION; }

}  // extern "C"
