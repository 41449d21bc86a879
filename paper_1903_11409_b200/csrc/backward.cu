// backward.cu — Batched SpMM backward.
//
// "The Batched SpMM is also applied to backward propagation."
// For C_i = A_i B_i and an upstream gradient G = dL/dC (same layout as C):
//   dL/dB_i   = A_i^T G_i           -> per-matrix transpose + the forward kernel
//   dL/dval_e = <G[row_e], B[col_e]> (SDDMM at A's sparsity pattern)
// (the standard adjoints).
//
// * transpose: one CTA per matrix expands its entries to (col, row) pairs
//   (position = storage position), and the stable device COO->CSR
//   (coo2csr.cu) sorts them, so A^T comes out in canonical (row, col,
//   original position) order, bit-exact against the oracle.
// * SDDMM: one CTA per matrix, a warp per row; each lane holds 128-bit
//   chunks of G's row, multiplies B's row chunks for every entry and the warp
//   reduces with shuffles (fixed butterfly order: deterministic).
#include <cstdint>

#include "internal.h"
#include "ptx.cuh"

namespace bspmm {

constexpr int kBwdThreads = 256;

// A_i entries -> (col, row) pairs at the same storage positions; nnz_off[i] = row_ptr[row_off[i]]
__global__ void __launch_bounds__(kBwdThreads) transpose_expand_kernel(int32_t batch, const int64_t* __restrict__ row_off,
                                                                       const int32_t* __restrict__ sizes,
                                                                       const int32_t* __restrict__ row_ptr,
                                                                       const int32_t* __restrict__ col,
                                                                       int32_t* __restrict__ idx,
                                                                       int64_t* __restrict__ nnz_off) {
  for (int64_t i = blockIdx.x; i < batch; i += gridDim.x) {
    const int64_t g0 = row_off[i];
    const int32_t n = sizes ? sizes[i] : (int32_t)(row_off[i + 1] - g0);
    if (threadIdx.x == 0) {
      nnz_off[i] = row_ptr[g0];
      if (i == batch - 1) nnz_off[batch] = row_ptr[g0 + n];
    }
    for (int32_t r = threadIdx.x >> 5; r < n; r += blockDim.x >> 5) {
      const int32_t e0 = row_ptr[g0 + r], e1 = row_ptr[g0 + r + 1];
      for (int32_t e = e0 + (threadIdx.x & 31); e < e1; e += 32) {
        idx[2 * (int64_t)e] = col[e];
        idx[2 * (int64_t)e + 1] = r;
      }
    }
  }
}

cudaError_t launch_transpose_expand(int32_t batch, const int64_t* row_off, const int32_t* sizes,
                                    const int32_t* row_ptr, const int32_t* col, int32_t* idx, int64_t* nnz_off,
                                    cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  const int grid = batch < 65535 ? batch : 65535;
  transpose_expand_kernel<<<grid, kBwdThreads, 0, s>>>(batch, row_off, sizes, row_ptr, col, idx, nnz_off);
  return cudaGetLastError();
}

// out[e] = sum_c G[row_e][c] * B[col_e][c]; VEC: float4 chunks (k, ldb, ldg % 4 == 0, aligned)
template <bool VEC>
__global__ void __launch_bounds__(kBwdThreads) sddmm_kernel(int32_t batch, int32_t k, const int64_t* __restrict__ row_off,
                                                           const int32_t* __restrict__ sizes,
                                                           const int32_t* __restrict__ row_ptr,
                                                           const int32_t* __restrict__ col,
                                                           const float* __restrict__ B, int64_t ldb,
                                                           const float* __restrict__ G, int64_t ldg,
                                                           float* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  constexpr int FW = VEC ? 4 : 1;
  const int32_t chunks = VEC ? (k >> 2) : k;
  constexpr int R = 8;  // G-row chunks a lane keeps in registers (k <= 32 * R * FW)
  for (int64_t i = blockIdx.x; i < batch; i += gridDim.x) {
    const int64_t g0 = row_off[i];
    const int32_t n = sizes ? sizes[i] : (int32_t)(row_off[i + 1] - g0);
    const float* Bi = B + g0 * ldb;
    for (int32_t r = warp; r < n; r += nw) {
      const float* grow = G + (g0 + r) * ldg;
      const int32_t e0 = row_ptr[g0 + r], e1 = row_ptr[g0 + r + 1];
      if (e1 == e0) continue;
      float4 gv[R];
      const bool inreg = chunks <= 32 * R;
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int32_t c = lane + 32 * q;
        gv[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (inreg && c < chunks) {
          if (VEC) gv[q] = ldg_nc_f4(grow + 4 * c);
          else gv[q].x = __ldg(grow + c);
        }
      }
      for (int32_t e = e0; e < e1; ++e) {
        const float* brow = Bi + (int64_t)__ldg(col + e) * ldb;
        float part = 0.f;
        if (inreg) {
#pragma unroll
          for (int q = 0; q < R; ++q) {
            const int32_t c = lane + 32 * q;
            if (c < chunks) {
              if (VEC) {
                const float4 b = ldg_nc_f4(brow + 4 * c);
                part = fmaf(gv[q].x, b.x, part);
                part = fmaf(gv[q].y, b.y, part);
                part = fmaf(gv[q].z, b.z, part);
                part = fmaf(gv[q].w, b.w, part);
              } else {
                part = fmaf(gv[q].x, __ldg(brow + c), part);
              }
            }
          }
        } else {
          for (int32_t c = lane; c < chunks; c += 32) {
            if (VEC) {
              const float4 a = ldg_nc_f4(grow + 4 * c), b = ldg_nc_f4(brow + 4 * c);
              part = fmaf(a.x, b.x, part);
              part = fmaf(a.y, b.y, part);
              part = fmaf(a.z, b.z, part);
              part = fmaf(a.w, b.w, part);
            } else {
              part = fmaf(__ldg(grow + c), __ldg(brow + c), part);
            }
          }
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(0xffffffffu, part, d);
        if (lane == 0) out[e] = part;
      }
    }
    (void)FW;
  }
}

cudaError_t launch_sddmm(int32_t batch, int32_t k, const int64_t* row_off, const int32_t* sizes,
                         const int32_t* row_ptr, const int32_t* col, const float* B, int64_t ldb, const float* G,
                         int64_t ldg, float* out, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  const int grid = batch < 65535 ? batch : 65535;
  const bool vec = (k % 4 == 0) && (ldb % 4 == 0) && (ldg % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(G)) & 15u) == 0;
  if (vec)
    sddmm_kernel<true><<<grid, kBwdThreads, 0, s>>>(batch, k, row_off, sizes, row_ptr, col, B, ldb, G, ldg, out);
  else
    sddmm_kernel<false><<<grid, kBwdThreads, 0, s>>>(batch, k, row_off, sizes, row_ptr, col, B, ldb, G, ldg, out);
  return cudaGetLastError();
}

}  // namespace bspmm
