// offsets.cu — batch-offset builder (hot-path row a-1) and the BSPMM_VALIDATE
// index checks.
//
// The paper builds the list of per-matrix pointers on the host and copies it
// host->device inside the timed region; at small n_B
// that copy decides the race against cuBLAS (:359).  Here the offsets are an
// int64 exclusive scan of the sizes computed on the device: one CTA of 1024
// threads, loads of 4 tiles in flight, warp-shuffle block scan per tile.
#include <cstdint>

#include "internal.h"

namespace bspmm {

constexpr int kScanThreads = 1024;
constexpr int kScanTiles = 4;  // tiles of 1024 sizes loaded before scanning

__global__ void __launch_bounds__(kScanThreads) offsets_kernel(int32_t batch, const int32_t* __restrict__ sizes,
                                                               int64_t* __restrict__ out) {
  __shared__ int64_t warp_tot[32];
  __shared__ int64_t carry_s;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) {
    carry_s = 0;
    out[0] = 0;
  }
  __syncthreads();
  for (int64_t base = 0; base < batch; base += (int64_t)kScanThreads * kScanTiles) {
    int32_t v[kScanTiles];
#pragma unroll
    for (int q = 0; q < kScanTiles; ++q) {
      const int64_t idx = base + (int64_t)q * kScanThreads + t;
      v[q] = idx < batch ? __ldg(sizes + idx) : 0;
    }
#pragma unroll
    for (int q = 0; q < kScanTiles; ++q) {
      // inclusive warp scan
      int64_t x = v[q];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
      }
      if (lane == 31) warp_tot[w] = x;
      __syncthreads();
      if (w == 0) {
        int64_t s = warp_tot[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int64_t y = __shfl_up_sync(0xffffffffu, s, d);
          if (lane >= d) s += y;
        }
        warp_tot[lane] = s;  // inclusive over warps
      }
      __syncthreads();
      const int64_t carry = carry_s;
      const int64_t incl = carry + (w ? warp_tot[w - 1] : 0) + x;
      const int64_t idx = base + (int64_t)q * kScanThreads + t;
      if (idx < batch) out[idx + 1] = incl;
      __syncthreads();
      if (t == kScanThreads - 1) carry_s = incl;
      __syncthreads();
    }
  }
}

cudaError_t launch_offsets(int32_t batch, const int32_t* sizes, int64_t* out, cudaStream_t s) {
  offsets_kernel<<<1, kScanThreads, 0, s>>>(batch, sizes, out);
  return cudaGetLastError();
}

// ---- BSPMM_VALIDATE ---------------------------------------------------------
__global__ void validate_sizes_kernel(int32_t batch, const int32_t* sizes, int* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < batch; i += (int64_t)gridDim.x * blockDim.x)
    if (sizes[i] < 0) atomicOr(flag, 1);
}

// per matrix: offsets monotone, n_i >= 0, row_ptr monotone on the matrix's rows, 0 <= col < n_i
__global__ void validate_csr_kernel(int32_t batch, const int64_t* row_off, const int32_t* sizes,
                                    const int32_t* row_ptr, const int32_t* col, int* flag) {
  for (int64_t i = blockIdx.x; i < batch; i += gridDim.x) {
    const int64_t g0 = row_off[i], g1 = row_off[i + 1];
    const int64_t n = sizes ? sizes[i] : g1 - g0;
    if (g0 < 0 || n < 0 || g0 + n > g1) {
      if (threadIdx.x == 0) atomicOr(flag, 2);
      continue;
    }
    for (int64_t r = threadIdx.x; r < n; r += blockDim.x) {
      const int32_t e0 = row_ptr[g0 + r], e1 = row_ptr[g0 + r + 1];
      if (e0 < 0 || e1 < e0) {
        atomicOr(flag, 4);
        continue;
      }
      for (int32_t e = e0; e < e1; ++e)
        if (col[e] < 0 || col[e] >= n) atomicOr(flag, 8);
    }
  }
}

__global__ void validate_coo_kernel(int32_t batch, const int64_t* row_off, const int32_t* sizes,
                                    const int64_t* nnz_off, const int32_t* idx, int* flag) {
  for (int64_t i = blockIdx.x; i < batch; i += gridDim.x) {
    const int64_t g0 = row_off[i], g1 = row_off[i + 1];
    const int64_t n = sizes ? sizes[i] : g1 - g0;
    const int64_t z0 = nnz_off[i], z1 = nnz_off[i + 1];
    if (g0 < 0 || n < 0 || g0 + n > g1 || z0 < 0 || z1 < z0) {
      if (threadIdx.x == 0) atomicOr(flag, 16);
      continue;
    }
    for (int64_t e = z0 + threadIdx.x; e < z1; e += blockDim.x) {
      const int32_t r = idx[2 * e], c = idx[2 * e + 1];
      if (r < 0 || r >= n || c < 0 || c >= n) atomicOr(flag, 32);
    }
  }
}

static int vgrid(int32_t batch) { return batch < 1 ? 1 : (batch < 4096 ? batch : 4096); }

cudaError_t launch_validate_sizes(int32_t batch, const int32_t* sizes, int* flag, cudaStream_t s) {
  validate_sizes_kernel<<<vgrid((batch + 255) / 256), 256, 0, s>>>(batch, sizes, flag);
  return cudaGetLastError();
}
cudaError_t launch_validate_csr(int32_t batch, const int64_t* row_off, const int32_t* sizes,
                                const int32_t* row_ptr, const int32_t* col, int* flag, cudaStream_t s) {
  validate_csr_kernel<<<vgrid(batch), 128, 0, s>>>(batch, row_off, sizes, row_ptr, col, flag);
  return cudaGetLastError();
}
cudaError_t launch_validate_coo(int32_t batch, const int64_t* row_off, const int32_t* sizes,
                                const int64_t* nnz_off, const int32_t* idx, int* flag, cudaStream_t s) {
  validate_coo_kernel<<<vgrid(batch), 128, 0, s>>>(batch, row_off, sizes, nnz_off, idx, flag);
  return cudaGetLastError();
}

}  // namespace bspmm
