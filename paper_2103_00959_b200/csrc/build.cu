// build.cu -- a1 COO -> canonical CSR of A~ = A + fill*I and a2 degree +
// symmetric normalisation (§4 Graph Notations, P:244
// Eq. gcn_layer, P:646 CSR design; readings A1-A8).
//
// Build pipeline (all hand-written kernels, one host sync at the end):
//   1. make_keys   slot t -> 64-bit key row*n + col (EMPTY = n*n for a missing
//                  reverse of a self-pair / invalid input), value = t.  Slots
//                  are laid out in the oracle's "pos" order (2i, 2i+1, loops),
//                  validation flags are OR-ed into a device word.
//   2. LSD radix   stable 8-bit passes over the bits of n*n: per-tile digit
//                  histogram, exclusive scan (digit-major), stable scatter
//                  (warp __match_any_sync ranking).  Stability keeps equal
//                  (row, col) keys in pos order.
//   3. coalesce    head flags -> exclusive scan -> per-head fp64 weight sum in
//                  pos order, one rounding to fp32.
//   4. row_ptr     gap-filling from the row changes of the sorted heads.
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace gsp {

constexpr int kRadixThreads = 256;
constexpr int kRadixItems = 8;
constexpr int64_t kRadixTile = kRadixThreads * kRadixItems;  // 2048 keys per tile
constexpr int64_t kScanTile = 2048;

enum : uint32_t { kErrRange = 1u, kErrNeg = 2u, kErrNonfinite = 4u };

static size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// ----------------------------------------------------------------- scan
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Block-wide exclusive scan of 2048 uint32 (8 per thread, blocked layout).
// If `sums` != NULL the tile total goes to sums[blockIdx.x]; if `offs` != NULL
// offs[blockIdx.x] is added to every output; out == NULL skips the outputs
// (reduce-only pass).  in may equal out (each thread reads before writing).
__global__ void __launch_bounds__(256) scan_tile_kernel(const uint32_t *in, uint32_t *out, int64_t L, uint32_t *sums,
                                                        const uint32_t *offs) {
  __shared__ uint32_t warp_tot[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)tid * 8;
  uint32_t v[8];
  uint32_t tsum = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i] = (base + i < L) ? in[base + i] : 0u;
    tsum += v[i];
  }
  uint32_t x = tsum;  // inclusive warp scan of thread sums
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  uint32_t wpre = 0, total = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    if (w < warp) wpre += warp_tot[w];
    total += warp_tot[w];
  }
  uint32_t run = wpre + x - tsum + (offs ? offs[blockIdx.x] : 0u);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t t = v[i];
    if (out && base + i < L) out[base + i] = run;
    run += t;
  }
  if (sums && tid == 0) sums[blockIdx.x] = total;
}

size_t scan_ws_bytes(int64_t L) {
  size_t b = 0;
  while (L > kScanTile) {
    L = ceil_div(L, kScanTile);
    b += align256((size_t)L * 4);
  }
  return b + 256;
}

// Exclusive scan of L uint32 (in may equal out); ws from scan_ws_bytes(L).
gsp_status scan_exclusive(const uint32_t *in, uint32_t *out, int64_t L, uint8_t *ws, cudaStream_t s) {
  if (L <= 0) return GSP_OK;
  const int64_t nt = ceil_div(L, kScanTile);
  if (nt == 1) {
    scan_tile_kernel<<<1, 256, 0, s>>>(in, out, L, nullptr, nullptr);
    return check_launch("scan_tile");
  }
  uint32_t *sums = reinterpret_cast<uint32_t *>(ws);
  uint8_t *rest = ws + align256((size_t)nt * 4);
  // pass 1: tile totals only; pass 2: scan with the scanned totals as offsets
  scan_tile_kernel<<<(unsigned)nt, 256, 0, s>>>(in, nullptr, L, sums, nullptr);
  gsp_status st = check_launch("scan_tile(up)");
  if (st) return st;
  st = scan_exclusive(sums, sums, nt, rest, s);
  if (st) return st;
  scan_tile_kernel<<<(unsigned)nt, 256, 0, s>>>(in, out, L, nullptr, sums);
  return check_launch("scan_tile(down)");
}

// ----------------------------------------------------------------- radix
__global__ void __launch_bounds__(kRadixThreads) radix_hist_kernel(const uint64_t *__restrict__ keys, int64_t N,
                                                                   int shift, uint32_t *__restrict__ counts,
                                                                   int64_t ntiles) {
  __shared__ uint32_t h[256];
  const int tid = threadIdx.x;
  h[tid] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRadixTile;
  if (base + kRadixTile <= N) {  // full tile: 16-byte loads (2 keys), all issued before the atomics
    ulonglong2 kv[kRadixItems / 2];
#pragma unroll
    for (int i = 0; i < kRadixItems / 2; ++i)
      kv[i] = *reinterpret_cast<const ulonglong2 *>(keys + base + 2 * ((int64_t)i * kRadixThreads + tid));
#pragma unroll
    for (int i = 0; i < kRadixItems / 2; ++i) {
      atomicAdd(&h[(unsigned)(kv[i].x >> shift) & 255u], 1u);
      atomicAdd(&h[(unsigned)(kv[i].y >> shift) & 255u], 1u);
    }
  } else {
#pragma unroll
    for (int i = 0; i < kRadixItems; ++i) {
      const int64_t k = base + (int64_t)i * kRadixThreads + tid;
      if (k < N) atomicAdd(&h[(unsigned)(keys[k] >> shift) & 255u], 1u);
    }
  }
  __syncthreads();
  counts[(int64_t)tid * ntiles + blockIdx.x] = h[tid];
}

__global__ void __launch_bounds__(kRadixThreads) radix_scatter_kernel(
    const uint64_t *__restrict__ kin, const uint32_t *__restrict__ vin, uint64_t *__restrict__ kout,
    uint32_t *__restrict__ vout, int64_t N, int shift, const uint32_t *__restrict__ offsets, int64_t ntiles) {
  __shared__ uint32_t wcnt[8][256];
  __shared__ uint32_t gbase[256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int w = 0; w < 8; ++w) wcnt[w][tid] = 0;
  gbase[tid] = offsets[(int64_t)tid * ntiles + blockIdx.x];
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRadixTile + (int64_t)warp * (32 * kRadixItems);
  uint64_t k[kRadixItems];
  uint32_t v[kRadixItems], rank[kRadixItems];
  int dig[kRadixItems];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < kRadixItems; ++i) {
    const int64_t idx = base + i * 32 + lane;
    const bool valid = idx < N;
    k[i] = valid ? kin[idx] : 0ull;
    v[i] = valid ? vin[idx] : 0u;
    const int d = valid ? (int)((k[i] >> shift) & 255u) : 256;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t before = 0;
    if (valid) before = wcnt[warp][d];
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) wcnt[warp][d] += __popc(peers);
    __syncwarp();
    rank[i] = before + __popc(peers & lt);
    dig[i] = d;
  }
  __syncthreads();
  uint32_t total;  // this tile's count of digit tid
  {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint32_t t = wcnt[w][tid];
      wcnt[w][tid] = run;
      run += t;
    }
    total = run;
  }
  // tile-local bucket starts: exclusive scan of the 256 digit totals
  __shared__ uint32_t tb[256];
  __shared__ uint32_t wsum[8];
  uint32_t incl = total;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  uint32_t wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += wsum[w];
  tb[tid] = wpre + incl - total;
  __syncthreads();
  // stage the tile in shared memory in output order (same positions as a
  // direct scatter: stable), then write each digit's run contiguously
  __shared__ uint64_t sk[kRadixTile];
  __shared__ uint32_t sv[kRadixTile];
#pragma unroll
  for (int i = 0; i < kRadixItems; ++i) {
    if (dig[i] < 256) {
      const uint32_t lpos = tb[dig[i]] + wcnt[warp][dig[i]] + rank[i];
      sk[lpos] = k[i];
      sv[lpos] = v[i];
    }
  }
  __syncthreads();
  const int64_t tile0 = (int64_t)blockIdx.x * kRadixTile;
  const int cnt = (int)min((int64_t)kRadixTile, N - tile0);
  for (int j = tid; j < cnt; j += kRadixThreads) {
    const uint64_t key = sk[j];
    const int d = (int)((key >> shift) & 255u);
    const uint32_t pos = gbase[d] + (uint32_t)j - tb[d];
    kout[pos] = key;
    vout[pos] = sv[j];
  }
}

// ----------------------------------------------------------------- build
template <typename IT>
__global__ void make_keys_kernel(int64_t n, int64_t m, const IT *__restrict__ src, const IT *__restrict__ dst,
                                 const float *__restrict__ w, int und, int with_loops, uint64_t *__restrict__ keys,
                                 uint32_t *__restrict__ vals, uint32_t *__restrict__ err) {
  // one thread per input pair i (both slots 2i, 2i + 1 of an undirected pair
  // in one 16-byte key store and one 8-byte value store), then one per loop
  const int64_t mm = und ? 2 * m : m;
  const int64_t T = m + (with_loops ? n : 0);
  const uint64_t EMPTY = (uint64_t)n * (uint64_t)n;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    if (t < m) {
      const int64_t u = (int64_t)src[t], v = (int64_t)dst[t];
      const uint32_t er = (u < 0 || u >= n || v < 0 || v >= n) ? kErrRange : 0u;
      uint32_t ef = er;  // the forward slot also validates the weight
      if (w) {
        const float wi = w[t];
        if (!isfinite(wi)) ef |= kErrNonfinite;
        else if (wi < 0.0f) ef |= kErrNeg;
      }
      if (ef) atomicOr(err, ef);
      const uint64_t kf = ef ? EMPTY : (uint64_t)u * n + v;
      if (und) {
        const uint64_t kr = (er || u == v) ? EMPTY : (uint64_t)v * n + u;  // reverse of a self pair: none
        *reinterpret_cast<ulonglong2 *>(keys + 2 * t) = make_ulonglong2(kf, kr);
        *reinterpret_cast<uint2 *>(vals + 2 * t) = make_uint2((uint32_t)(2 * t), (uint32_t)(2 * t + 1));
      } else {
        keys[t] = kf;
        vals[t] = (uint32_t)t;
      }
    } else {
      const uint64_t u = (uint64_t)(t - m);
      keys[mm + (int64_t)u] = u * n + u;
      vals[mm + (int64_t)u] = (uint32_t)(mm + (int64_t)u);
    }
  }
}

__global__ void head_flags_kernel(const uint64_t *__restrict__ keys, int64_t S, uint64_t EMPTY,
                                  uint32_t *__restrict__ head) {
  // 4 keys per thread (two 16-byte loads, one 16-byte store of the flags)
  for (int64_t k = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); k < S;
       k += 4 * (int64_t)gridDim.x * blockDim.x) {
    if (k + 4 <= S) {
      const ulonglong2 a = *reinterpret_cast<const ulonglong2 *>(keys + k);
      const ulonglong2 b = *reinterpret_cast<const ulonglong2 *>(keys + k + 2);
      const uint64_t p = k ? keys[k - 1] : ~0ull;
      uint4 f;
      f.x = (a.x < EMPTY && (k == 0 || p != a.x)) ? 1u : 0u;
      f.y = (a.y < EMPTY && a.x != a.y) ? 1u : 0u;
      f.z = (b.x < EMPTY && a.y != b.x) ? 1u : 0u;
      f.w = (b.y < EMPTY && b.x != b.y) ? 1u : 0u;
      *reinterpret_cast<uint4 *>(head + k) = f;
    } else {
      for (int64_t j = k; j < S; ++j) {
        const uint64_t key = keys[j];
        head[j] = (key < EMPTY && (j == 0 || keys[j - 1] != key)) ? 1u : 0u;
      }
    }
  }
}

// For every head: fp64 sum of the run's weights in pos order -> fp32; the
// column; and the row_ptr entries of rows that start here (gap filling).
// key / n for key < n^2, n < 2^31 without the 64-bit division subroutine:
// a double-precision estimate (off by at most one) corrected exactly
__device__ __forceinline__ uint64_t div_by_n(uint64_t key, uint64_t n, double inv_n) {
  uint64_t r = (uint64_t)((double)key * inv_n);
  if (r * n > key) --r;
  else if ((r + 1) * n <= key) ++r;
  return r;
}

__global__ void coalesce_kernel(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ pos, int64_t S,
                                int64_t n, int64_t m, int und, const float *__restrict__ w, float fill,
                                const uint32_t *__restrict__ head, const uint32_t *__restrict__ idx,
                                int64_t *__restrict__ row_ptr, int32_t *__restrict__ col, float *__restrict__ val,
                                int64_t *__restrict__ nnz_out) {
  // 4 consecutive sorted slots per thread: keys / head / idx / pos by 16-byte
  // loads, each key's row computed once (the previous slot's row carried)
  const uint64_t EMPTY = (uint64_t)n * (uint64_t)n;
  const int64_t mm = und ? 2 * m : m;
  const double inv_n = 1.0 / (double)n;
  for (int64_t k0 = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); k0 < S;
       k0 += 4 * (int64_t)gridDim.x * blockDim.x) {
    uint64_t kk[5];  // keys k0 .. k0 + 3 and k0 + 4 (EMPTY past the end)
    uint32_t hd[4], ix[4];
    if (k0 + 4 <= S) {
      const ulonglong2 a = *reinterpret_cast<const ulonglong2 *>(keys + k0);
      const ulonglong2 b = *reinterpret_cast<const ulonglong2 *>(keys + k0 + 2);
      kk[0] = a.x, kk[1] = a.y, kk[2] = b.x, kk[3] = b.y;
      const uint4 h = *reinterpret_cast<const uint4 *>(head + k0);
      const uint4 x = *reinterpret_cast<const uint4 *>(idx + k0);
      hd[0] = h.x, hd[1] = h.y, hd[2] = h.z, hd[3] = h.w;
      ix[0] = x.x, ix[1] = x.y, ix[2] = x.z, ix[3] = x.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        kk[q] = k0 + q < S ? keys[k0 + q] : EMPTY;
        hd[q] = k0 + q < S ? head[k0 + q] : 0u;
        ix[q] = k0 + q < S ? idx[k0 + q] : 0u;
      }
    }
    kk[4] = k0 + 4 < S ? keys[k0 + 4] : EMPTY;
    int64_t prev_r = (k0 == 0) ? -1 : (int64_t)div_by_n(keys[k0 - 1], (uint64_t)n, inv_n);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t k = k0 + q;
      const uint64_t key = kk[q];
      if (k >= S || key >= EMPTY) break;  // sorted: EMPTY keys only at the end
      const bool last_valid = kk[q + 1] >= EMPTY;
      const int64_t r = (int64_t)div_by_n(key, (uint64_t)n, inv_n);
      if (hd[q]) {
        double sum = 0.0;
        for (int64_t j = k; j < S && keys[j] == key; ++j) {
          const int64_t p = pos[j];
          double wj;
          if (p < mm) {
            const int64_t i = und ? (p >> 1) : p;
            wj = w ? (double)w[i] : 1.0;
          } else {
            wj = (double)fill;
          }
          sum = __dadd_rn(sum, wj);
        }
        const int64_t o = ix[q];
        col[o] = (int32_t)(key - (uint64_t)r * n);
        val[o] = __double2float_rn(sum);
        for (int64_t rr = prev_r + 1; rr <= r; ++rr) row_ptr[rr] = o;
      }
      if (last_valid) {
        const int64_t total = (int64_t)ix[q] + hd[q];
        for (int64_t rr = r + 1; rr <= n; ++rr) row_ptr[rr] = total;
        *nnz_out = total;
      }
      prev_r = r;
    }
  }
}

__global__ void fill_i64_kernel(int64_t *p, int64_t count, int64_t v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// Stable LSD radix sort of (key, value) pairs on the low `bits` bits of the
// keys, 8 bits per pass, ping-ponging between the two buffer pairs; on
// return keys/vals point at the sorted arrays.  counts: radix_counts_bytes(N),
// scan_ws: radix_scan_ws_bytes(N).
size_t radix_counts_bytes(int64_t N) { return (size_t)256 * std::max<int64_t>(1, ceil_div(N, kRadixTile)) * 4; }
size_t radix_scan_ws_bytes(int64_t N) { return scan_ws_bytes(256 * std::max<int64_t>(1, ceil_div(N, kRadixTile))); }
gsp_status radix_sort_pairs(uint64_t *&keys, uint32_t *&vals, uint64_t *keys_alt, uint32_t *vals_alt, int64_t N,
                            int bits, uint32_t *counts, uint8_t *scan_ws, cudaStream_t s) {
  const int64_t ntiles = ceil_div(N, kRadixTile);
  uint64_t *ka = keys, *kb = keys_alt;
  uint32_t *va = vals, *vb = vals_alt;
  gsp_status st = GSP_OK;
  for (int shift = 0; shift < bits; shift += 8) {
    radix_hist_kernel<<<(unsigned)ntiles, kRadixThreads, 0, s>>>(ka, N, shift, counts, ntiles);
    if ((st = check_launch("radix_hist"))) return st;
    if ((st = scan_exclusive(counts, counts, 256 * ntiles, scan_ws, s))) return st;  // digit-major offsets
    radix_scatter_kernel<<<(unsigned)ntiles, kRadixThreads, 0, s>>>(ka, va, kb, vb, N, shift, counts, ntiles);
    if ((st = check_launch("radix_scatter"))) return st;
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  keys = ka;
  vals = va;
  return GSP_OK;
}

struct BuildLayout {
  size_t keys_a, keys_b, vals_a, vals_b, counts, head, idx, scan, scalars, total;
};

static int key_bits(int64_t n) {
  const unsigned __int128 e = (unsigned __int128)n * (unsigned __int128)n;  // EMPTY
  int b = 0;
  while (b < 127 && (((unsigned __int128)1) << b) <= e) ++b;
  return std::max(b, 1);
}

static BuildLayout build_layout(int64_t S) {
  BuildLayout L{};
  const int64_t ntiles = std::max<int64_t>(1, ceil_div(S, kRadixTile));
  size_t off = 0;
  auto take = [&](size_t b) {
    const size_t o = off;
    off += align256(std::max<size_t>(b, 1));
    return o;
  };
  L.keys_a = take((size_t)S * 8);
  L.keys_b = take((size_t)S * 8);
  L.vals_a = take((size_t)S * 4);
  L.vals_b = take((size_t)S * 4);
  L.counts = take((size_t)256 * ntiles * 4);
  L.head = take((size_t)S * 4);
  L.idx = take((size_t)S * 4);
  L.scan = take(std::max(scan_ws_bytes(256 * ntiles), scan_ws_bytes(S)));
  L.scalars = take(64);
  L.total = off;
  return L;
}

static int64_t slots(int64_t n, int64_t m, uint32_t flags, float fill) {
  return ((flags & GSP_UNDIRECTED) ? 2 * m : m) + (fill != 0.0f ? n : 0);
}

// ----------------------------------------------------------------- normalise
// d_u = sum of row u's values in fp64 (P:244 D~_ii = sum_j A~_ij) and
// a_uv = fp32(w / sqrt(d_u d_v)) with IEEE RN fp64 ops (A8).  One warp per row
// (8 rows per CTA); rows longer than kNormLong entries are handled by the
// whole CTA after its short rows.  Degree order: lane-strided fp64 partials,
// xor tree, then (long rows) the 8 warps in order -- fixed per row, and equal
// to the oracle's sequential sum whenever the row sum is exact in fp64 (every
// integer / dyadic weight; DESIGN.md §3 A8).
constexpr int kNormLong = 1024;

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// d_u = sum of row u's values in fp64.  A CTA owns 32 rows (4 per warp), their
// extents staged in shared memory; a warp issues the first 32-entry batch of
// all four rows before reducing any (lane l adds entries l, l + 32, ... of a
// row in order, then an xor tree -- the per-row order of one warp per row);
// rows of more than kNormLong entries are reduced afterwards by the whole CTA
// (thread t adds entries t, t + 256, ..., xor tree per warp, warps in order).
constexpr int kDegRows = 32;
__global__ void __launch_bounds__(256) degree_kernel(const int64_t *__restrict__ rp, const float *__restrict__ val,
                                                     int64_t n, double *__restrict__ deg) {
  __shared__ int64_t s_rp[kDegRows + 1];
  __shared__ int s_long[kDegRows];
  __shared__ int s_nlong;
  __shared__ double s_part[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * kDegRows;
  const int nr = (int)min((int64_t)kDegRows, n - r0);
  if (tid == 0) s_nlong = 0;
  if (tid <= nr) s_rp[tid] = __ldg(rp + r0 + tid);
  __syncthreads();
  float v0[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // first batch of the warp's four rows, all in flight
    const int j = warp * 4 + q;
    const int64_t b = j < nr ? s_rp[j] : 0, e1 = j < nr ? s_rp[j + 1] : 0;
    v0[q] = (j < nr && e1 - b <= kNormLong && b + lane < e1) ? __ldg(val + b + lane) : 0.0f;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int j = warp * 4 + q;
    if (j >= nr) break;
    const int64_t b = s_rp[j], e1 = s_rp[j + 1];
    if (e1 - b > kNormLong) {
      if (lane == 0) s_long[atomicAdd(&s_nlong, 1)] = j;
      continue;
    }
    double sum = 0.0;
    if (b + lane < e1) sum += (double)v0[q];
#pragma unroll 4
    for (int64_t e = b + lane + 32; e < e1; e += 32) sum += (double)__ldg(val + e);
    sum = warp_sum_f64(sum);
    if (lane == 0) deg[r0 + j] = sum;
  }
  __syncthreads();
  for (int k = 0; k < s_nlong; ++k) {
    const int64_t r = r0 + s_long[k];
    const int64_t b = s_rp[s_long[k]], e1 = s_rp[s_long[k] + 1];
    double sum = 0.0;
#pragma unroll 4
    for (int64_t e = b + tid; e < e1; e += 256) sum += (double)__ldg(val + e);
    sum = warp_sum_f64(sum);
    if (lane == 0) s_part[warp] = sum;
    __syncthreads();
    if (tid == 0) {
      double t = s_part[0];
      for (int w = 1; w < 8; ++w) t += s_part[w];
      deg[r] = t;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ float norm_entry(double du, double dv, float w) {
  const double p = __dmul_rn(du, dv);
  double r = 0.0;
  if (p != 0.0) {
    const double q = __dsqrt_rn(p);
    // unit weights (every benchmark graph): the correctly rounded reciprocal
    // is exactly the correctly rounded 1 / q, and cheaper than the division
    r = (w == 1.0f) ? __drcp_rn(q) : __ddiv_rn((double)w, q);
  }
  return __double2float_rn(r);
}

// One launch, two kinds of CTA (long ones first, so the power-law tail
// overlaps the bulk):
//  * LONG CTA c scans rows [256 c, 256 c + 256) (one coalesced load of their
//    extents), collects the rows of more than kNormLong entries in shared
//    memory and normalises each with the whole CTA, 4 entries per thread per
//    round (every load of a round issued before the arithmetic);
//  * SHORT CTA b owns rows [32 b, 32 b + 32): their entries are contiguous,
//    so the CTA walks them edge-parallel (coalesced col / val loads, 4 per
//    thread per round), finds each entry's row by a binary search of the 33
//    staged row pointers and skips entries of long rows.
// Each value depends on (d_u, d_v, w) only: bit-identical to any schedule.
constexpr int kNormSlice = 256;  // rows scanned by a long CTA
constexpr int kNormRows = 32;    // rows of a short CTA
__global__ void __launch_bounds__(256) normalize_kernel(const int64_t *__restrict__ rp,
                                                        const int32_t *__restrict__ col, const float *val,
                                                        int64_t n, const double *__restrict__ deg, float *val_out,
                                                        int n_long) {
  const int tid = threadIdx.x;
  if ((int)blockIdx.x < n_long) {
    __shared__ int s_long[kNormSlice];
    __shared__ int s_n;
    const int64_t r0 = (int64_t)blockIdx.x * kNormSlice;
    if (tid == 0) s_n = 0;
    __syncthreads();
    const int64_t r = r0 + tid;
    if (r < n && __ldg(rp + r + 1) - __ldg(rp + r) > kNormLong) s_long[atomicAdd(&s_n, 1)] = tid;
    __syncthreads();
    const int nl = s_n;
    for (int k = 0; k < nl; ++k) {
      const int64_t u = r0 + s_long[k];
      const int64_t b = __ldg(rp + u), e1 = __ldg(rp + u + 1);
      const double du = __ldg(deg + u);
      for (int64_t e0 = b + tid; e0 < e1; e0 += 4 * 256) {
        int c[4];
        float w[4];
        double dv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t e = e0 + 256 * q;
          c[q] = e < e1 ? __ldg(col + e) : 0;
          w[q] = e < e1 ? val[e] : 0.0f;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) dv[q] = e0 + 256 * q < e1 ? __ldg(deg + c[q]) : 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t e = e0 + 256 * q;
          if (e < e1) val_out[e] = norm_entry(du, dv[q], w[q]);
        }
      }
    }
    return;
  }
  __shared__ int64_t s_rp[kNormRows + 1];
  __shared__ double s_du[kNormRows];
  const int64_t r0 = (int64_t)(blockIdx.x - n_long) * kNormRows;
  const int nr = (int)min((int64_t)kNormRows, n - r0);
  if (tid <= nr) s_rp[tid] = __ldg(rp + r0 + tid);
  if (tid < nr) s_du[tid] = __ldg(deg + r0 + tid);
  __syncthreads();
  const int64_t E0 = s_rp[0], E1 = s_rp[nr];
  const int lane = tid & 31;
  // lane l holds the start of row l + 1 (rows 1 .. nr - 1; later lanes: never
  // <= an entry).  The row of entry e is #{j >= 1 : s_rp[j] <= e}: a warp's 32
  // consecutive entries c .. c + 31 start from row(c) = one ballot, then each
  // lane steps forward over the (few) rows starting inside the chunk
  const int64_t start_l = lane + 1 < nr ? s_rp[lane + 1] : INT64_MAX;
  // warp-uniform loop (every lane reaches the ballots): warp w takes the
  // 32-entry chunks E0 + 32 w + 256 k
  for (int64_t wb = E0 + (tid & ~31); wb < E1; wb += 4 * 256) {
    const int64_t e0 = wb + lane;
    int c[4], row[4];
    float w[4];
    double dv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t e = e0 + 256 * q;
      const int64_t cw = wb + 256 * q;  // the chunk's first entry (warp-uniform)
      int j = __popc(__ballot_sync(0xffffffffu, start_l <= cw));
      if (e < E1) {
        while (j + 1 < nr && s_rp[j + 1] <= e) ++j;
        if (s_rp[j + 1] - s_rp[j] > kNormLong) j = -1;
      } else {
        j = -1;
      }
      row[q] = j;
      c[q] = j >= 0 ? __ldg(col + e) : 0;
      w[q] = j >= 0 ? val[e] : 0.0f;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) dv[q] = row[q] >= 0 ? __ldg(deg + c[q]) : 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (row[q] >= 0) val_out[e0 + 256 * q] = norm_entry(s_du[row[q]], dv[q], w[q]);
  }
}

}  // namespace gsp

using namespace gsp;

extern "C" gsp_status gsp_coo_to_csr_workspace(int64_t n, int64_t m, uint32_t flags, float fill, size_t *ws_bytes,
                                               int64_t *nnz_max) {
  clear_detail();
  if (n < 0 || m < 0 || !ws_bytes) return fail(GSP_ERR_INVALID_ARG, "gsp_coo_to_csr_workspace: bad argument");
  if (n >= (int64_t(1) << 31)) return fail(GSP_ERR_UNSUPPORTED, "n must be < 2^31");
  const int64_t S = slots(n, m, flags, fill);
  if (S >= (int64_t(1) << 32) - 1) return fail(GSP_ERR_UNSUPPORTED, "2m + n must be < 2^32");
  *ws_bytes = build_layout(S).total;
  if (nnz_max) *nnz_max = S;
  return GSP_OK;
}

extern "C" gsp_status gsp_coo_to_csr(int64_t n, int64_t m, const void *src, const void *dst, gsp_index_type it,
                                     const float *w, uint32_t flags, float fill, int64_t *row_ptr, int32_t *col_idx,
                                     float *val, int64_t *nnz_out, void *ws, size_t ws_bytes, gsp_stream stream) {
  const char *fn = "gsp_coo_to_csr";
  clear_detail();
  if (n < 0 || m < 0) return fail(GSP_ERR_INVALID_ARG, "%s: negative size", fn);
  if (n >= (int64_t(1) << 31)) return fail(GSP_ERR_UNSUPPORTED, "%s: n must be < 2^31", fn);
  if (it != GSP_I32 && it != GSP_I64) return fail(GSP_ERR_INVALID_ARG, "%s: bad index type", fn);
  if (!std::isfinite(fill)) return fail(GSP_ERR_NONFINITE, "%s: fill is not finite", fn);
  if (fill < 0.0f) return fail(GSP_ERR_NEGATIVE_WEIGHT, "%s: fill < 0", fn);
  if (!row_ptr || !nnz_out) return fail(GSP_ERR_INVALID_ARG, "%s: row_ptr / nnz_out is NULL", fn);
  if (m > 0 && (!src || !dst)) return fail(GSP_ERR_INVALID_ARG, "%s: src / dst is NULL", fn);
  if (m > 0 && n == 0) return fail(GSP_ERR_INDEX_RANGE, "%s: edges on an empty node set", fn);
  const int und = (flags & GSP_UNDIRECTED) ? 1 : 0;
  const int64_t S = slots(n, m, flags, fill);
  if (S >= (int64_t(1) << 32) - 1) return fail(GSP_ERR_UNSUPPORTED, "%s: 2m + n must be < 2^32", fn);
  if (S > 0 && (!col_idx || !val)) return fail(GSP_ERR_INVALID_ARG, "%s: col_idx / val is NULL", fn);
  const BuildLayout Lw = build_layout(S);
  if (!ws || ws_bytes < Lw.total) return fail(GSP_ERR_WORKSPACE, "%s: workspace needs %zu bytes", fn, Lw.total);
  if (reinterpret_cast<uintptr_t>(ws) & 255u) return fail(GSP_ERR_WORKSPACE, "%s: ws must be 256-byte aligned", fn);
  cudaStream_t s = cs(stream);
  uint8_t *W = reinterpret_cast<uint8_t *>(ws);
  if (S == 0) {
    fill_i64_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n + 1, 256), 4096)), 256, 0, s>>>(
        row_ptr, n + 1, 0);
    gsp_status st = check_launch("fill_row_ptr");
    if (!st) *nnz_out = 0;
    return st;
  }
  uint64_t *ka = reinterpret_cast<uint64_t *>(W + Lw.keys_a), *kb = reinterpret_cast<uint64_t *>(W + Lw.keys_b);
  uint32_t *va = reinterpret_cast<uint32_t *>(W + Lw.vals_a), *vb = reinterpret_cast<uint32_t *>(W + Lw.vals_b);
  uint32_t *counts = reinterpret_cast<uint32_t *>(W + Lw.counts);
  uint32_t *head = reinterpret_cast<uint32_t *>(W + Lw.head), *idx = reinterpret_cast<uint32_t *>(W + Lw.idx);
  uint8_t *scan_ws = W + Lw.scan;
  uint32_t *d_err = reinterpret_cast<uint32_t *>(W + Lw.scalars);
  int64_t *d_nnz = reinterpret_cast<int64_t *>(W + Lw.scalars + 8);

  if (cudaMemsetAsync(W + Lw.scalars, 0, 16, s) != cudaSuccess) return check_launch("memset");
  const unsigned gb = (unsigned)std::min<int64_t>(ceil_div(S, 256), 65535 * 4);
  const unsigned gk = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(m + n, 256), 65535 * 4));
  const unsigned gh = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(S, 4 * 256), 65535 * 4));
  if (it == GSP_I32)
    make_keys_kernel<int32_t><<<gk, 256, 0, s>>>(n, m, (const int32_t *)src, (const int32_t *)dst, w, und,
                                                 fill != 0.0f, ka, va, d_err);
  else
    make_keys_kernel<int64_t><<<gk, 256, 0, s>>>(n, m, (const int64_t *)src, (const int64_t *)dst, w, und,
                                                 fill != 0.0f, ka, va, d_err);
  gsp_status st = check_launch("make_keys");
  if (st) return st;

  // stable LSD radix sort over the bits of EMPTY = n*n
  if ((st = radix_sort_pairs(ka, va, kb, vb, S, key_bits(n), counts, scan_ws, s))) return st;
  const uint64_t EMPTY = (uint64_t)n * (uint64_t)n;
  head_flags_kernel<<<gh, 256, 0, s>>>(ka, S, EMPTY, head);
  if ((st = check_launch("head_flags"))) return st;
  if ((st = scan_exclusive(head, idx, S, scan_ws, s))) return st;
  fill_i64_kernel<<<1, 256, 0, s>>>(row_ptr, 1, 0);  // row_ptr[0] = 0 even if row 0 is empty
  coalesce_kernel<<<gh, 256, 0, s>>>(ka, va, S, n, m, und, w, fill, head, idx, row_ptr, col_idx, val, d_nnz);
  if ((st = check_launch("coalesce"))) return st;

  struct {
    uint32_t err, pad;
    int64_t nnz;
  } h{};
  if (cudaMemcpyAsync(&h, W + Lw.scalars, 16, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return check_launch("sync");
  if (h.err & kErrRange) return fail(GSP_ERR_INDEX_RANGE, "%s: an endpoint is outside [0, n)", fn);
  if (h.err & kErrNonfinite) return fail(GSP_ERR_NONFINITE, "%s: non-finite weight", fn);
  if (h.err & kErrNeg) return fail(GSP_ERR_NEGATIVE_WEIGHT, "%s: negative weight", fn);
  *nnz_out = h.nnz;
  return GSP_OK;
}

extern "C" gsp_status gsp_sym_normalize_workspace(const gsp_csr *a, size_t *ws_bytes) {
  clear_detail();
  if (!a || !ws_bytes || a->n_rows < 0) return fail(GSP_ERR_INVALID_ARG, "gsp_sym_normalize_workspace: bad argument");
  *ws_bytes = (size_t)a->n_rows * sizeof(double);
  return GSP_OK;
}

extern "C" gsp_status gsp_sym_normalize(const gsp_csr *a, float *val_out, double *deg_out, void *ws, size_t ws_bytes,
                                        gsp_stream stream) {
  const char *fn = "gsp_sym_normalize";
  clear_detail();
  gsp_status st = check_csr(a, true, fn);
  if (st) return st;
  if (a->n_rows != a->n_cols) return fail(GSP_ERR_INVALID_ARG, "%s: matrix must be square", fn);
  if (a->n_rows == 0) return GSP_OK;
  if (a->nnz > 0 && !val_out) return fail(GSP_ERR_INVALID_ARG, "%s: val_out is NULL", fn);
  if (val_out && val_out != a->val && overlaps(val_out, (size_t)a->nnz * 4, a->val, (size_t)a->nnz * 4))
    return fail(GSP_ERR_ALIAS, "%s: val_out partially overlaps val", fn);
  double *d = deg_out;
  if (!d) {  // the degrees go to the caller's workspace (the library never allocates)
    if (!ws || ws_bytes < (size_t)a->n_rows * sizeof(double) || !aligned8(ws))
      return fail(GSP_ERR_WORKSPACE, "%s: deg_out is NULL: an 8-byte aligned workspace of %zu bytes is required", fn,
                  (size_t)a->n_rows * sizeof(double));
    d = static_cast<double *>(ws);
  }
  if (val_out && overlaps(val_out, (size_t)a->nnz * 4, d, (size_t)a->n_rows * 8))
    return fail(GSP_ERR_ALIAS, "%s: val_out overlaps the degree array", fn);
  cudaStream_t s = cs(stream);
  const unsigned gb = (unsigned)ceil_div(a->n_rows, kDegRows);
  degree_kernel<<<gb, 256, 0, s>>>(a->row_ptr, a->val, a->n_rows, d);
  if ((st = check_launch("degree"))) return st;
  if (a->nnz == 0) return GSP_OK;
  const int64_t n_long = ceil_div(a->n_rows, kNormSlice);
  normalize_kernel<<<(unsigned)(n_long + ceil_div(a->n_rows, kNormRows)), 256, 0, s>>>(
      a->row_ptr, a->col_idx, a->val, a->n_rows, d, val_out, (int)n_long);
  return check_launch("normalize");
}
