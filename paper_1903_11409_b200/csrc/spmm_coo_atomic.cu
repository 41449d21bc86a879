// spmm_coo_atomic.cu — the paper's SWA SpMM for SparseTensor (SURVEY §8(f)
// NEXT-3): PAPER.md:162-165 and Fig. algo:code_swa_spmm_st (lines 175-185),
// with the output tile in shared memory (Fig. batched_spmm_algo (a)/(b),
// PAPER.md:218-226) and one thread block per (SpMM op, column block)
// (PAPER.md:254-257).
//
// A sub-warp of L lanes takes one nonzero (rid, cid, val) of the UNSORTED
// SparseTensor; lane l adds val * B[cid][j] into the shared C
// tile for the tile's columns j = l, l + L, ... (128-bit chunks here) with
// shared-memory atomics, exactly the paper's Atomic(C[rid][j] += val *
// B[cid][j]) (:184).  The C tile is zeroed in shared memory first (no init
// launch, :220-222) and written back coalesced.  Atomic accumulation order is
// not deterministic: results are checked against the north_star bound only
// (the deterministic path is bspmm_coo = COO->CSR + the CSR kernel).
//
// B200 choices: the B tile is staged with one TMA bulk copy when it is the
// whole contiguous B_i (else read through L1); the unit's metadata is a
// single round trip (nnz_off and row_off only: the SparseTensor needs no
// row pointers).
#include <cstdint>

#include "internal.h"
#include "ptx.cuh"

namespace bspmm {

constexpr int kStThreads = 256;

struct StParams {
  int64_t units;
  int32_t tiles, kt, k, lanes, cap_rows;
  const int64_t* row_off;
  const int32_t* sizes;
  const int64_t* nnz_off;
  const int2* idx;
  const float* vals;
  const float* B;
  int64_t ldb;
  float* C;
  int64_t ldc;
};

__device__ __forceinline__ const float* bsrc_of(const StParams& p, int64_t g0, int32_t c0) {
  return p.B + g0 * p.ldb + c0;
}

__global__ void __launch_bounds__(kStThreads) spmm_coo_atomic_kernel(const StParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  const int64_t u = blockIdx.x;
  const int64_t i = u / p.tiles;
  const int32_t t = (int32_t)(u - i * p.tiles);
  const int64_t g0 = p.row_off[i];
  const int32_t n = p.sizes ? p.sizes[i] : (int32_t)(p.row_off[i + 1] - g0);
  const int64_t z0 = p.nnz_off[i], z1 = p.nnz_off[i + 1];
  const int32_t c0 = t * p.kt, kw = min(p.kt, p.k - c0), kw4 = kw >> 2;
  if (n == 0) return;
  float* Cg = p.C + g0 * p.ldc + c0;
  const int L = p.lanes;
  const int lane = threadIdx.x & 31, li = lane % L;
  const int64_t group = (threadIdx.x / L), ngroups = blockDim.x / L;
  if (n > p.cap_rows) {
    // case 3: no shared-memory tile; zero C, then atomics in global memory
    for (int32_t q = threadIdx.x; q < n * kw4; q += blockDim.x) {
      const int32_t r = q / kw4, c = q - r * kw4;
      *reinterpret_cast<float4*>(Cg + (int64_t)r * p.ldc + 4 * c) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    for (int64_t e = z0 + group; e < z1; e += ngroups) {
      const int2 rc = p.idx[e];
      const float v = p.vals[e];
      for (int32_t c = li; c < kw4; c += L) {
        const float4 b = ldg_nc_f4(bsrc_of(p, g0, c0) + (int64_t)rc.y * p.ldb + 4 * c);
        float* dst = Cg + (int64_t)rc.x * p.ldc + 4 * c;
        atomicAdd(dst + 0, v * b.x);
        atomicAdd(dst + 1, v * b.y);
        atomicAdd(dst + 2, v * b.z);
        atomicAdd(dst + 3, v * b.w);
      }
    }
    return;
  }
  float4* Cs = reinterpret_cast<float4*>(smem);                          // n x kw4
  const bool staged = kw == p.ldb;                                        // whole contiguous B_i
  float4* Bs = Cs + (size_t)p.cap_rows * (p.kt >> 2);                     // n x kw4 (staged case)
  const float* bsrc = bsrc_of(p, g0, c0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (staged && threadIdx.x == 0) {
    const uint32_t tx = (uint32_t)n * (uint32_t)kw * 4u;
    mbar_arrive_expect_tx(&bar, tx);
    bulk_g2s(Bs, bsrc, tx, &bar);
  }
  // set C to O in shared memory while B lands
  for (int32_t q = threadIdx.x; q < n * kw4; q += blockDim.x) Cs[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  if (staged) mbar_wait(&bar, 0);
  for (int64_t e = z0 + group; e < z1; e += ngroups) {
    const int2 rc = p.idx[e];  // (rid, cid)
    const float v = p.vals[e];
    float4* crow = Cs + (size_t)rc.x * kw4;
    for (int32_t c = li; c < kw4; c += L) {
      const float4 b = staged ? Bs[(size_t)rc.y * kw4 + c] : ldg_nc_f4(bsrc + (int64_t)rc.y * p.ldb + 4 * c);
      float* dst = reinterpret_cast<float*>(crow + c);
      atomicAdd(dst + 0, v * b.x);
      atomicAdd(dst + 1, v * b.y);
      atomicAdd(dst + 2, v * b.z);
      atomicAdd(dst + 3, v * b.w);
    }
  }
  __syncthreads();
  for (int32_t q = threadIdx.x; q < n * kw4; q += blockDim.x) {
    const int32_t r = q / kw4, c = q - r * kw4;
    stg_cs_f4(Cg + (int64_t)r * p.ldc + 4 * c, Cs[q]);
  }
}

// smem budget: C tile + (staged) B tile, for up to cap_rows rows
cudaError_t launch_spmm_coo_atomic(int32_t batch, int32_t k, const int64_t* row_off, const int32_t* sizes,
                                   const int64_t* nnz_off, const int32_t* idx, const float* vals, const float* B,
                                   int64_t ldb, float* C, int64_t ldc, int32_t max_rows, int32_t smem_optin,
                                   cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  // column block so that the C tile of the largest matrix fits
  const int32_t R = max_rows > 0 ? max_rows : 64;
  int32_t kt = align_up(k, 4);
  while ((int64_t)R * kt * 4 * 2 > smem_optin - 2048 && kt > 4) kt = align_up(kt / 2, 4);
  const int32_t kt4 = kt / 4;
  StParams p;
  p.tiles = (int32_t)ceil_div(k, kt);
  p.units = (int64_t)batch * p.tiles;
  p.kt = kt;
  p.k = k;
  p.lanes = pow2_ceil(kt4 < 32 ? kt4 : 32);  // the paper's subWarp rule on float4 chunks
  p.cap_rows = R;
  p.row_off = row_off;
  p.sizes = sizes;
  p.nnz_off = nnz_off;
  p.idx = reinterpret_cast<const int2*>(idx);
  p.vals = vals;
  p.B = B;
  p.ldb = ldb;
  p.C = C;
  p.ldc = ldc;
  const int smem = 2 * R * kt4 * 16;
  if (smem > 47 * 1024) {  // dynamic + static above the 48 KB default
    cudaError_t e = cudaFuncSetAttribute(spmm_coo_atomic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  if (p.units > 0x7fffffffLL) return cudaErrorInvalidValue;
  spmm_coo_atomic_kernel<<<(unsigned)p.units, kStThreads, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace bspmm
