// coo2csr.cu — device COO/SparseTensor -> canonical CSR (hot-path row a-2).
//
// The paper multiplies unsorted SparseTensor entries directly with atomics
// (SWA-ST, Fig. algo:code_swa_spmm_st; unsorted :141).  This
// build converts on the device first so that the result is deterministic and
// the CSR is bit-exact against the oracle (R5/R15):
//   key(e) = (row << 32) | col for entry e of matrix i, stable-sorted, so
//   equal (row, col) keep their input order (duplicates are summed later in
//   that order, as PAPER.md:101 accumulates them).
// One CTA per matrix.  The sort is a bottom-up merge sort in which every
// element finds its output slot by binary search in the sibling run
// ("merge by rank": left elements count right keys < x, right elements count
// left keys <= x, which is exactly stable).  It runs in shared memory when the
// matrix has at most `cap` entries, otherwise in a global-memory workspace
// (same algorithm, so the same order).  The row pointer is then
// row_ptr[g0 + r] = nnz_off[i] + lower_bound(keys, r << 32).
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
  for (int64_t i = blockIdx.x; i < batch; i += gridDim.x) {
    const int64_t g0 = row_off[i], g1 = row_off[i + 1];
    const int32_t n = sizes ? sizes[i] : (int32_t)(g1 - g0);
    const int64_t z0 = nnz_off[i];
    const int32_t m = (int32_t)(nnz_off[i + 1] - z0);
    uint64_t *k0, *k1;
    uint32_t *p0, *p1;
    if (m <= cap) {
      k0 = reinterpret_cast<uint64_t*>(smem);
      k1 = k0 + cap;
      p0 = reinterpret_cast<uint32_t*>(k1 + cap);
      p1 = p0 + cap;
    } else {
      k0 = ws_keys + z0;
      k1 = ws_keys + ws_stride + z0;
      p0 = ws_pay + z0;
      p1 = ws_pay + ws_stride + z0;
    }
    const int2* pairs = reinterpret_cast<const int2*>(idx) + z0;
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
    __syncthreads();  // smem reuse by the next matrix of this CTA
  }
}

int32_t coo_smem_cap(int64_t max_nnz_hint, int32_t smem_optin) {
  const int64_t per = 2 * (8 + 4);  // two key + payload buffers
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
  const int smem = cap * 2 * (8 + 4);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(coo2csr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  const int grid = batch < 65535 ? batch : 65535;
  coo2csr_kernel<<<grid, kCooThreads, smem, s>>>(batch, row_off, sizes, nnz_off, idx, vals, row_ptr, col_out,
                                                  val_out, ws_keys, ws_pay, ws_stride, cap);
  return cudaGetLastError();
}

}  // namespace bspmm
