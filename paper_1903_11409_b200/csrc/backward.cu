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
#include <algorithm>
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

// Staged SDDMM (float4 path, k <= 512): each CTA walks matrices; B_i lands in
// shared memory with one TMA bulk copy (per-row copies when ldb > k), a warp
// per row keeps its grad_C row in registers and forms two dot products per
// iteration from shared memory (independent loads first), reduced across the
// warp with a fixed butterfly (deterministic).  Matrices whose B_i exceeds
// the capacity read B from global memory in the same loop.
template <int CH, bool STAGED>
__device__ __forceinline__ void sddmm_rows(int32_t n, int32_t chunks, const float* __restrict__ Bsrc, int64_t bld,
                                           const float* __restrict__ Grow0, int64_t ldg,
                                           const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                           float* __restrict__ out, int lane, int warp, int nw) {
  // rows r = warp, warp + nw, ...; the next row's grad_C chunks and row range
  // are loaded while the current row computes (one exposed latency per matrix)
  float4 gn[CH];
  int32_t n0 = 0, n1 = 0;
  bool ok[CH];
#pragma unroll
  for (int v = 0; v < CH; ++v) ok[v] = lane + 32 * v < chunks;
  auto gload = [&](int32_t r_, float4* dst) {
    const float* grow = Grow0 + (int64_t)r_ * ldg;
#pragma unroll
    for (int v = 0; v < CH; ++v) dst[v] = ok[v] ? ldg_nc_f4(grow + 4 * (lane + 32 * v)) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  if (warp < n) {
    n0 = __ldg(rp + warp);
    n1 = __ldg(rp + warp + 1);
    gload(warp, gn);
  }
  for (int32_t r = warp; r < n; r += nw) {
    const int32_t e0 = n0, e1 = n1;
    float4 gv[CH];
#pragma unroll
    for (int v = 0; v < CH; ++v) gv[v] = gn[v];
    if (r + nw < n) {
      n0 = __ldg(rp + r + nw);
      n1 = __ldg(rp + r + nw + 1);
      gload(r + nw, gn);
    }
    if (e1 == e0) continue;
    auto bload = [&](int32_t cc, int v) -> float4 {
      const float* q = Bsrc + (int64_t)cc * bld + 4 * (lane + 32 * v);
      return STAGED ? *reinterpret_cast<const float4*>(q) : ldg_nc_f4(q);
    };
    int32_t e = e0;
    for (; e + 1 < e1; e += 2) {
      const int32_t c0 = __ldg(col + e), c1 = __ldg(col + e + 1);
      float4 b0[CH], b1[CH];
#pragma unroll
      for (int v = 0; v < CH; ++v) {
        if (ok[v]) {
          b0[v] = bload(c0, v);
          b1[v] = bload(c1, v);
        }
      }
      float p0 = 0.f, p1 = 0.f;
#pragma unroll
      for (int v = 0; v < CH; ++v) {
        if (ok[v]) {
          p0 = fmaf(gv[v].x, b0[v].x, p0); p0 = fmaf(gv[v].y, b0[v].y, p0);
          p0 = fmaf(gv[v].z, b0[v].z, p0); p0 = fmaf(gv[v].w, b0[v].w, p0);
          p1 = fmaf(gv[v].x, b1[v].x, p1); p1 = fmaf(gv[v].y, b1[v].y, p1);
          p1 = fmaf(gv[v].z, b1[v].z, p1); p1 = fmaf(gv[v].w, b1[v].w, p1);
        }
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        p0 += __shfl_xor_sync(0xffffffffu, p0, d);
        p1 += __shfl_xor_sync(0xffffffffu, p1, d);
      }
      if (lane == 0) {
        out[e] = p0;
        out[e + 1] = p1;
      }
    }
    if (e < e1) {
      const int32_t c0 = __ldg(col + e);
      float p0 = 0.f;
#pragma unroll
      for (int v = 0; v < CH; ++v) {
        if (ok[v]) {
          const float4 b = bload(c0, v);
          p0 = fmaf(gv[v].x, b.x, p0); p0 = fmaf(gv[v].y, b.y, p0);
          p0 = fmaf(gv[v].z, b.z, p0); p0 = fmaf(gv[v].w, b.w, p0);
        }
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) p0 += __shfl_xor_sync(0xffffffffu, p0, d);
      if (lane == 0) out[e] = p0;
    }
  }
}

template <int CH>
__global__ void __launch_bounds__(kBwdThreads) sddmm_staged_kernel(int32_t batch, int32_t k,
                                                                  const int64_t* __restrict__ row_off,
                                                                  const int32_t* __restrict__ sizes,
                                                                  const int32_t* __restrict__ row_ptr,
                                                                  const int32_t* __restrict__ col,
                                                                  const float* __restrict__ B, int64_t ldb,
                                                                  const float* __restrict__ G, int64_t ldg,
                                                                  float* __restrict__ out, int32_t cap_bytes) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  float* Bs = reinterpret_cast<float*>(smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int32_t chunks = k >> 2;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t phase = 0;
  for (int64_t i = blockIdx.x; i < batch; i += gridDim.x) {
    const int64_t g0 = row_off[i];
    const int32_t n = sizes ? sizes[i] : (int32_t)(row_off[i + 1] - g0);
    const bool staged = n > 0 && (int64_t)n * k * 4 <= cap_bytes;
    if (staged) {
      if (threadIdx.x == 0) {
        const uint32_t bytes = (uint32_t)n * (uint32_t)k * 4u;
        mbar_arrive_expect_tx(&bar, bytes);
        if (ldb == k) {
          bulk_g2s(Bs, B + g0 * ldb, bytes, &bar);
        } else {
          for (int32_t r = 0; r < n; ++r) bulk_g2s(Bs + (int64_t)r * k, B + (g0 + r) * ldb, (uint32_t)k * 4u, &bar);
        }
      }
      mbar_wait(&bar, phase);
      phase ^= 1u;
      sddmm_rows<CH, true>(n, chunks, Bs, k, G + g0 * ldg, ldg, row_ptr + g0, col, out, lane, warp, nw);
    } else {
      sddmm_rows<CH, false>(n, chunks, B + g0 * ldb, ldb, G + g0 * ldg, ldg, row_ptr + g0, col, out, lane, warp,
                            nw);
    }
    __syncthreads();  // every warp is done with Bs before the next matrix's copy
  }
}

cudaError_t launch_sddmm(int32_t batch, int32_t k, const int64_t* row_off, const int32_t* sizes,
                         const int32_t* row_ptr, const int32_t* col, const float* B, int64_t ldb, const float* G,
                         int64_t ldg, float* out, int32_t max_rows_hint, int32_t num_sms, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  const bool vec = (k % 4 == 0) && (ldb % 4 == 0) && (ldg % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(G)) & 15u) == 0;
  if (vec && k <= 512) {
    // capacity: the hinted largest matrix (3 CTAs per SM fit up to ~72 KB each)
    constexpr int32_t kCapMax = 72 * 1024;
    int32_t cap = kCapMax;
    if (max_rows_hint > 0 && (int64_t)max_rows_hint * k * 4 < kCapMax) cap = (int32_t)max_rows_hint * k * 4;
    cap = (cap + 127) & ~127;
    const int grid = (int)std::min<int64_t>(batch, (int64_t)num_sms * 8);
    cudaError_t e = cudaSuccess;
    const int chunks = k >> 2, ch = (chunks + 31) / 32;
    auto go = [&](auto kern) {
      if (cap > 48 * 1024) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
        if (e != cudaSuccess) return;
      }
      kern<<<grid, kBwdThreads, cap, s>>>(batch, k, row_off, sizes, row_ptr, col, B, ldb, G, ldg, out, cap);
      e = cudaGetLastError();
    };
    if (ch <= 1) go(sddmm_staged_kernel<1>);
    else if (ch <= 2) go(sddmm_staged_kernel<2>);
    else go(sddmm_staged_kernel<4>);
    return e;
  }
  const int grid = batch < 65535 ? batch : 65535;
  if (vec)
    sddmm_kernel<true><<<grid, kBwdThreads, 0, s>>>(batch, k, row_off, sizes, row_ptr, col, B, ldb, G, ldg, out);
  else
    sddmm_kernel<false><<<grid, kBwdThreads, 0, s>>>(batch, k, row_off, sizes, row_ptr, col, B, ldb, G, ldg, out);
  return cudaGetLastError();
}

}  // namespace bspmm
