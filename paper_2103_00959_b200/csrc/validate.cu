// validate.cu -- GSP_VALIDATE mode: non-finite logits / attention inputs are
// rejected with GSP_ERR_NONFINITE before any compute launch (SPEC.md S:164-166
// "pre: all finite ... errors: non-finite logit"; SURVEY §8(b) "Non-finite
// logits are checked only under GSP_VALIDATE"; reading A12).
//
// The mode is per calling thread (gsp_set_flags); validating calls check their
// logit-like inputs with one streaming kernel each and synchronise their
// stream once to read the verdict.  The verdict word is a __device__ array in
// the library image (no runtime allocation); validating calls on one device
// are serialised by a host mutex so concurrent threads never share a word.
#include <mutex>

#include "common.cuh"

namespace gsp {

static thread_local uint32_t g_flags = 0;

__device__ unsigned int g_nonfinite[64];  // one word per device ordinal

__global__ void nonfinite_kernel(const uint32_t *__restrict__ p, int64_t n, int dev) {
  unsigned int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    bad |= ((__ldg(p + i) & 0x7f800000u) == 0x7f800000u);  // exponent all ones: Inf or NaN
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(&g_nonfinite[dev], 1u);
}

bool validate_mode() { return (g_flags & GSP_VALIDATE) != 0; }

// Check arrays of fp32 values for NaN / Inf (count elements each, contiguous).
// Returns GSP_OK, GSP_ERR_NONFINITE (naming the array) or GSP_ERR_CUDA.
gsp_status check_finite(cudaStream_t s, const char *fn, int narr, const float *const *arr, const int64_t *count,
                        const char *const *name) {
  static std::mutex mu[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return fail(GSP_ERR_CUDA, "%s: no device", fn);
  std::lock_guard<std::mutex> lock(mu[dev]);
  const int grid = 2 * sm_count();
  for (int k = 0; k < narr; ++k) {
    if (!arr[k] || count[k] <= 0) continue;
    const unsigned int zero = 0;
    if (cudaMemcpyToSymbolAsync(g_nonfinite, &zero, sizeof(zero), dev * sizeof(unsigned int),
                                cudaMemcpyHostToDevice, s) != cudaSuccess)
      return check_launch("validate: reset");
    nonfinite_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const uint32_t *>(arr[k]), count[k], dev);
    gsp_status st = check_launch("validate: nonfinite_kernel");
    if (st) return st;
    unsigned int flag = 0;
    if (cudaMemcpyFromSymbolAsync(&flag, g_nonfinite, sizeof(flag), dev * sizeof(unsigned int),
                                  cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return check_launch("validate: read flag");
    if (flag) return fail(GSP_ERR_NONFINITE, "%s: %s holds a NaN or Inf (GSP_VALIDATE)", fn, name[k]);
  }
  return GSP_OK;
}

}  // namespace gsp

extern "C" gsp_status gsp_set_flags(uint32_t flags) {
  gsp::clear_detail();
  if (flags & ~uint32_t(GSP_VALIDATE)) return gsp::fail(GSP_ERR_INVALID_ARG, "gsp_set_flags: unknown flag bits");
  gsp::g_flags = flags;
  return GSP_OK;
}

extern "C" uint32_t gsp_get_flags(void) { return gsp::g_flags; }
