// coo2csr.cu — device COO/SparseTensor -> canonical CSR (hot-path row a-2).
//
// The paper multiplies unsorted SparseTensor entries directly with atomics
// (SWA-ST, Fig. algo:code_swa_spmm_st; unsorted :141).  This
// build converts on the device first so that the result is deterministic and
// the CSR is bit-exact against the oracle (R5/R15):
//   key(e) = (row << 32) | col for entry e of matrix i, stable-sorted, so
//   equal (row, col) keep their input order (duplicates are summed later in
//   that order, as PAPER.md:101 accumulates them).
// One CTA per matrix.  Shared-memory path (up to `cap` entries and rows): a
// counting sort by row (histogram, scan, scatter into row segments in any
// order), then each entry's slot in its segment is its rank by the unique key
// (col, original position) -- deterministic and canonical whatever the
// scatter order.  Larger matrices: a bottom-up merge sort in a global
// workspace in which every element finds its output slot by binary search in
// the sibling run ("merge by rank": left elements count right keys < x, right
// elements count left keys <= x, exactly stable), then
// row_ptr[g0 + r] = nnz_off[i] + lower_bound(keys, r << 32).  Both give the
// same (row, col, position) order.
#include <cstdint>

#include "internal.h"

namespace bspmm {

constexpr int kCooThreads = 256;

__device__ __forceinline__ int32_t lower_bound_u64(const uint64_t* a, int32_t n, uint64_t x) {
  int32_t lo = 0, hi = n;
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int32_t upper_bound_u64(const uint64_t* a, int32_t n, uint64_t x) {
  int32_t lo = 0, hi = n;
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// stable merge sort of keys[0..m) with payload; result in the returned buffer (0 or 1)
__device__ int merge_sort(uint64_t* k0, uint32_t* p0, uint64_t* k1, uint32_t* p1, int32_t m) {
  int cur = 0;
  for (int32_t w = 1; w < m; w <<= 1) {
    const uint64_t* ki = cur ? k1 : k0;
    const uint32_t* pi = cur ? p1 : p0;
    uint64_t* ko = cur ? k0 : k1;
    uint32_t* po = cur ? p0 : p1;
    for (int32_t q = threadIdx.x; q < m; q += blockDim.x) {
      const int32_t start = q / (2 * w) * (2 * w);
      const int32_t mid = min(start + w, m), end = min(start + 2 * w, m);
      const uint64_t x = ki[q];
      int32_t pos;
      if (q < mid) pos = (q - start) + lower_bound_u64(ki + mid, end - mid, x);
      else pos = (q - mid) + upper_bound_u64(ki + start, mid - start, x);
      ko[start + pos] = x;
      po[start + pos] = pi[q];
    }
    __syncthreads();
    cur ^= 1;
  }
  return cur;
}

// Shared-memory path (m <= cap entries, n <= cap rows): counting sort by row,
// then every entry finds its slot in its row segment by rank of the unique key
// (col, original position).  Scatter order inside a segment is arbitrary
// (shared atomics); the rank makes the result canonical and deterministic.
__device__ void coo2csr_small(const int2* __restrict__ pairs, const float* __restrict__ vals, int32_t m, int32_t n,
                              int64_t z0, int64_t g0, int64_t g1, bool last, int32_t* __restrict__ row_ptr,
                              int32_t* __restrict__ col_out, float* __restrict__ val_out, unsigned char* smem,
                              int32_t cap) {
  int32_t* sr = reinterpret_cast<int32_t*>(smem);  // row of entry e        [cap]
  int32_t* sc = sr + cap;                          // col of entry e        [cap]
  int32_t* slot = sc + cap;                        // segment slot -> e     [cap]
  int32_t* start = slot + cap;                     // row starts            [cap + 1]
  int32_t* cursor = start + cap + 1;               // per-row fill / counts [cap]
  __shared__ int32_t warp_tot[kCooThreads / 32];
  for (int32_t r = threadIdx.x; r < n; r += blockDim.x) cursor[r] = 0;
  __syncthreads();
  for (int32_t e = threadIdx.x; e < m; e += blockDim.x) {
    const int2 rc = pairs[e];
    sr[e] = rc.x;
    sc[e] = rc.y;
    atomicAdd(&cursor[rc.x], 1);
  }
  __syncthreads();
  // exclusive scan of the row counts (block-wide, chunked by blockDim)
  int32_t carry = 0;
  for (int32_t base = 0; base < n; base += blockDim.x) {
    const int32_t r = base + threadIdx.x;
    const int32_t v = r < n ? cursor[r] : 0;
    int32_t x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    int32_t wpre = 0, tot = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
      if (q < w) wpre += warp_tot[q];
      tot += warp_tot[q];
    }
    if (r < n) start[r] = carry + wpre + x - v;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) start[n] = m;
  for (int32_t r = threadIdx.x; r < n; r += blockDim.x) cursor[r] = 0;
  __syncthreads();
  for (int32_t e = threadIdx.x; e < m; e += blockDim.x) {
    const int32_t r = sr[e];
    slot[start[r] + atomicAdd(&cursor[r], 1)] = e;
  }
  __syncthreads();
  for (int32_t q = threadIdx.x; q < m; q += blockDim.x) {
    const int32_t e = slot[q];
    const int32_t r = sr[e], c = sc[e];
    const int32_t s0 = start[r], s1 = start[r + 1];
    int32_t rank = 0;
    for (int32_t t = s0; t < s1; ++t) {
      const int32_t f = slot[t];
      const int32_t cf = sc[f];
      rank += (cf < c) || (cf == c && f < e);
    }
    col_out[z0 + s0 + rank] = c;
    val_out[z0 + s0 + rank] = vals[e];  // bitwise move
  }
  for (int32_t r = threadIdx.x; r < n; r += blockDim.x) row_ptr[g0 + r] = (int32_t)(z0 + start[r]);
  for (int64_t g = g0 + n + threadIdx.x; g < g1; g += blockDim.x) row_ptr[g] = (int32_t)(z0 + m);
  if (last && threadIdx.x == 0) row_ptr[g1] = (int32_t)(z0 + m);
  __syncthreads();  // shared memory reuse by the CTA's next matrix
}

__global__ void __launch_bounds__(kCooThreads) coo2csr_kernel(int32_t batch, const int64_t* __restrict__ row_off,
                                                              const int32_t* __restrict__ sizes,
                                                              const int64_t* __restrict__ nnz_off,
                                                              const int32_t* __restrict__ idx,
                                                              const float* __restrict__ vals,
                                                              int32_t* __restrict__ row_ptr,
                                                              int32_t* __restrict__ col_out,
                                                              float* __restrict__ val_out, uint64_t* ws_keys,
                                                              uint32_t* ws_pay, int64_t ws_stride, int32_t cap) {
  extern __shared__ __align__(16) unsigned char smem[];
  // the SpMM that consumes this CSR is launched with programmatic stream
  // serialization: let its prologue start now (it waits for our completion
  // before touching memory)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int64_t i = blockIdx.x; i < batch; i += gridDim.x) {
    const int64_t g0 = row_off[i], g1 = row_off[i + 1];
    const int32_t n = sizes ? sizes[i] : (int32_t)(g1 - g0);
    const int64_t z0 = nnz_off[i];
    const int32_t m = (int32_t)(nnz_off[i + 1] - z0);
    const int2* pairs = reinterpret_cast<const int2*>(idx) + z0;
    if (m <= cap && n <= cap) {
      coo2csr_small(pairs, vals + z0, m, n, z0, g0, g1, i == batch - 1, row_ptr, col_out, val_out, smem, cap);
      continue;
    }
    // large matrix: stable merge sort of (row << 32 | col) keys in the global workspace
    uint64_t* k0 = ws_keys + z0;
    uint64_t* k1 = ws_keys + ws_stride + z0;
    uint32_t* p0 = ws_pay + z0;
    uint32_t* p1 = ws_pay + ws_stride + z0;
    for (int32_t q = threadIdx.x; q < m; q += blockDim.x) {
      const int2 rc = pairs[q];
      k0[q] = ((uint64_t)(uint32_t)rc.x << 32) | (uint32_t)rc.y;
      p0[q] = (uint32_t)q;
    }
    __syncthreads();
    const int which = merge_sort(k0, p0, k1, p1, m);
    const uint64_t* ks = which ? k1 : k0;
    const uint32_t* ps = which ? p1 : p0;
    for (int32_t q = threadIdx.x; q < m; q += blockDim.x) {
      col_out[z0 + q] = (int32_t)(uint32_t)(ks[q] & 0xffffffffu);
      val_out[z0 + q] = vals[z0 + ps[q]];  // bitwise move
    }
    for (int32_t r = threadIdx.x; r < n; r += blockDim.x)
      row_ptr[g0 + r] = (int32_t)(z0 + lower_bound_u64(ks, m, (uint64_t)(uint32_t)r << 32));
    for (int64_t g = g0 + n + threadIdx.x; g < g1; g += blockDim.x) row_ptr[g] = (int32_t)(z0 + m);
    if (i == batch - 1 && threadIdx.x == 0) row_ptr[g1] = (int32_t)(z0 + m);
    __syncthreads();
  }
}

int32_t coo_smem_cap(int64_t max_nnz_hint, int32_t smem_optin) {
  const int64_t per = 5 * 4;  // row, col, slot, start, cursor (int32) per entry / row
  int64_t cap = max_nnz_hint > 0 ? max_nnz_hint : kCooSmemCap;
  const int64_t lim = (smem_optin - 1024) / per;
  if (cap > lim) cap = lim;
  if (cap < 1) cap = 1;
  return (int32_t)cap;
}

cudaError_t launch_coo2csr(int32_t batch, const int64_t* row_off, const int32_t* sizes, const int64_t* nnz_off,
                           const int32_t* idx, const float* vals, int32_t* row_ptr, int32_t* col_out,
                           float* val_out, uint64_t* ws_keys, uint32_t* ws_pay, int64_t ws_stride, int32_t cap,
                           cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  const int smem = (5 * cap + 1) * 4;
  if (smem > 47 * 1024) {  // dynamic + static above the 48 KB default
    cudaError_t e = cudaFuncSetAttribute(coo2csr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  const int grid = batch < 65535 ? batch : 65535;
  coo2csr_kernel<<<grid, kCooThreads, smem, s>>>(batch, row_off, sizes, nnz_off, idx, vals, row_ptr, col_out,
                                                  val_out, ws_keys, ws_pay, ws_stride, cap);
  return cudaGetLastError();
}

}  // namespace bspmm
