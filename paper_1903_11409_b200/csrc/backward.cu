// backward.cu — Batched SpMM backward.
//
// "The Batched SpMM is also applied to backward propagation."
// For C_i = A_i B_i and an upstream gradient G = dL/dC (same layout as C):
//   dL/dB_i   = A_i^T G_i           -> per-matrix transpose + the forward kernel
//   dL/dval_e = <G[row_e], B[col_e]> (SDDMM at A's sparsity pattern)
// (the standard adjoints).
//
// * transpose: a stable counting sort of each matrix's entries by column
//   (counts, scan, then a scatter in storage order in which equal columns
//   rank by __match_any_sync), so A^T comes out in canonical (row, col,
//   original position) order, bit-exact against the oracle -- one warp per
//   matrix (transpose_csr_kernel; columns counted in windows of WIN, so any
//   n_i works), or, for small batches with hints, one CTA per matrix whose 8
//   warps split the entries (transpose_cta_kernel).
// * SDDMM: a warp per row; each lane holds 128-bit chunks of G's row,
//   multiplies B's row chunks (B_i staged in shared memory) for every entry
//   and the warp reduces with shuffles (fixed butterfly order: deterministic)
//   -- sddmm_struct_kernel (streaming batches: the CSR slice double-buffered
//   in shared memory by cp.async), sddmm_staged_kernel (the round-1 kernel,
//   k > 256), sddmm_kernel (unaligned / scalar).
// * backward_fused_kernel (streaming batches, both adjoints): grad_C_i staged
//   once feeds grad_B = A^T grad_C (A_i^T formed in shared memory) and the
//   SDDMM.
#include <algorithm>
#include <cstdint>

#include "internal.h"
#include "ptx.cuh"

namespace bspmm {

constexpr int kBwdThreads = 256;
// experiment bits (include/bspmm_debug.h): the standalone SDDMM with its
// structure read from global memory (the round-1 kernel); two grad_C rows
// prefetched instead of one
constexpr int32_t kDbgSddmmGlobalStruct = 1 << 27;
constexpr int32_t kDbgSddmmPf2 = 1 << 28;

// CSR -> per-matrix transposed CSR, one warp per matrix (see the header).
// Entries of A_i are visited in storage order = (row, position) order, so a
// stable counting sort by column yields A^T's canonical (row, col, position)
// order: rowT[g0 + c] = z0 + #entries with column < c, and an entry of column
// c goes to slot start[c] + #earlier entries of column c.
// Latency: a warp's global loads are issued together, never as a dependent
// chain -- the row-pointer slice lands in shared memory in one round trip (an
// entry's row is then a binary search there), and each block of 256 entries'
// columns and values land in registers (8 per lane) in one round trip, kept
// for the scatter when the matrix has <= 256 entries.
// Shared memory per warp: WIN column cursors, kTrRp row pointers and up to
// `ridcap` row ids (every entry's row, filled from the shared row pointers, so
// the scatter needs no search; above the capacity: binary search).
constexpr int kTrWarps = 8;
constexpr int kTrRp = 516;  // row-pointer slice capacity (n_i <= 515; larger: search in global memory)
constexpr int kTrE = 8;     // entries per lane per block (256-entry blocks)
template <int WIN>          // columns counted per window (WIN / 32 per lane)
__global__ void __launch_bounds__(kTrWarps * 32) transpose_csr_kernel(int32_t batch, const int64_t* __restrict__ row_off,
                                                                      const int32_t* __restrict__ sizes,
                                                                      const int32_t* __restrict__ row_ptr,
                                                                      const int32_t* __restrict__ col,
                                                                      const float* __restrict__ vals,
                                                                      int32_t* __restrict__ rowT,
                                                                      int32_t* __restrict__ colT,
                                                                      float* __restrict__ valsT, int32_t ridcap) {
  extern __shared__ __align__(16) int32_t tr_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int32_t* cnt = tr_smem + (size_t)w * (WIN + kTrRp + ridcap);
  int32_t* rps = cnt + WIN;
  int32_t* rid = rps + kTrRp;
  const uint32_t lt = (1u << lane) - 1u;
  for (int64_t i = (int64_t)blockIdx.x * kTrWarps + w; i < batch; i += (int64_t)gridDim.x * kTrWarps) {
    const int64_t g0 = row_off[i], g1 = row_off[i + 1];
    const int32_t n = sizes ? sizes[i] : (int32_t)(g1 - g0);
    const int32_t* rp = row_ptr + g0;
    const bool rp_s = n < kTrRp;
    if (rp_s) {
      int32_t t[(kTrRp + 31) / 32];
#pragma unroll
      for (int q = 0; q < (kTrRp + 31) / 32; ++q) {
        const int32_t r = lane + 32 * q;
        if (r <= n) t[q] = __ldg(rp + r);
      }
#pragma unroll
      for (int q = 0; q < (kTrRp + 31) / 32; ++q) {
        const int32_t r = lane + 32 * q;
        if (r <= n) rps[r] = t[q];
      }
      __syncwarp();
    }
    const int32_t z0 = rp_s ? rps[0] : __ldg(rp), z1 = rp_s ? rps[n] : __ldg(rp + n);
    const bool use_rid = rp_s && z1 - z0 <= ridcap;
    if (use_rid) {
      for (int32_t r = lane; r < n; r += 32)
        for (int32_t e = rps[r], e1 = rps[r + 1]; e < e1; ++e) rid[e - z0] = r;
      __syncwarp();
    }
    for (int64_t g = g0 + n + lane; g < g1; g += 32) rowT[g] = z1;  // padding rows: empty
    if (i == batch - 1 && lane == 0) rowT[g1] = row_ptr[g1];
    // one 256-entry block in registers: column ids (-1 past the end) and values
    int32_t cq[kTrE];
    float vq[kTrE];
    auto load_blk = [&](int32_t blk) {
#pragma unroll
      for (int q = 0; q < kTrE; ++q) {
        const int32_t e = blk + 32 * q + lane;
        cq[q] = e < z1 ? __ldg(col + e) : -1;
        vq[q] = e < z1 ? __ldg(vals + e) : 0.f;
      }
    };
    const bool resident = z1 - z0 <= 32 * kTrE;
    if (resident) load_blk(z0);
    int32_t before = 0;  // entries whose column precedes the window
    for (int32_t w0 = 0; w0 < n; w0 += WIN) {
      const int32_t wn = min(WIN, n - w0);
#pragma unroll
      for (int q = 0; q < WIN / 32; ++q) cnt[lane + 32 * q] = 0;
      __syncwarp();
      for (int32_t blk = z0; blk < z1; blk += 32 * kTrE) {
        if (!resident) load_blk(blk);
#pragma unroll
        for (int q = 0; q < kTrE; ++q) {
          const int32_t c = cq[q] - w0;
          if (cq[q] >= 0 && c >= 0 && c < wn) atomicAdd(&cnt[c], 1);
        }
      }
      __syncwarp();
      // exclusive scan of the window's counts: lane owns WIN/32 consecutive columns
      int32_t v[WIN / 32], sum = 0;
#pragma unroll
      for (int q = 0; q < WIN / 32; ++q) {
        v[q] = cnt[lane * (WIN / 32) + q];
        sum += v[q];
      }
      int32_t x = sum;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
      }
      int32_t run = before + x - sum;
#pragma unroll
      for (int q = 0; q < WIN / 32; ++q) {
        const int32_t c = lane * (WIN / 32) + q;
        cnt[c] = run;  // becomes the column's cursor (slot relative to z0)
        if (c < wn) rowT[g0 + w0 + c] = z0 + run;
        run += v[q];
      }
      before += __shfl_sync(0xffffffffu, x, 31);
      __syncwarp();
      // stable scatter, 32 entries at a time in storage order
      for (int32_t blk = z0; blk < z1; blk += 32 * kTrE) {
        if (!resident) load_blk(blk);
#pragma unroll
        for (int q = 0; q < kTrE; ++q) {
          const int32_t e = blk + 32 * q + lane;
          if (blk + 32 * q >= z1) break;  // warp-uniform
          const int32_t c = cq[q] >= 0 ? cq[q] - w0 : -1;
          const bool in = c >= 0 && c < wn;
          const uint32_t peers = __match_any_sync(0xffffffffu, in ? c : -1);
          if (in) {
            const int32_t slot = cnt[c] + __popc(peers & lt);
            // row of entry e: the last r with rp[r] <= e (empty rows share rp)
            int32_t lo = 0, hi = n - 1;
            if (use_rid) lo = hi = rid[e - z0];
            while (lo < hi) {
              const int32_t mid = (lo + hi + 1) >> 1;
              if ((rp_s ? rps[mid] : __ldg(rp + mid)) <= e) lo = mid;
              else hi = mid - 1;
            }
            colT[z0 + slot] = lo;
            valsT[z0 + slot] = vq[q];  // bitwise move
          }
          __syncwarp();
          if (in && (peers & lt) == 0) cnt[c] += __popc(peers);
          __syncwarp();
        }
      }
    }
  }
}

// CTA-per-matrix transpose for small (latency-bound) batches: the warp
// kernel above gives a whole matrix to one warp, so on C3 (200 matrices of
// up to 300 rows / 1370 entries) 25 SMs work and the largest matrix's serial
// passes set the time.  Here the 8 warps of a CTA split the matrix's entries
// into 8 contiguous ranges: each warp counts its range per column (32 entries
// at a time, equal columns grouped by __match_any_sync), a thread per column
// turns the 8 counts into per-warp offsets and the column total, warp 0 scans
// the totals into the A^T row pointers, and each warp scatters its range in
// storage order (slot = column start + the earlier warps' count + the running
// count within the warp) -- a stable counting sort: the same canonical order,
// the same bits.  Matrices above the (hinted) shared-memory capacities run a
// plain global-memory version of the same sort.
constexpr int kTcWarps = kBwdThreads / 32;
__global__ void __launch_bounds__(kBwdThreads) transpose_cta_kernel(int32_t batch, const int64_t* __restrict__ row_off,
                                                                   const int32_t* __restrict__ sizes,
                                                                   const int32_t* __restrict__ row_ptr,
                                                                   const int32_t* __restrict__ col,
                                                                   const float* __restrict__ vals,
                                                                   int32_t* __restrict__ rowT, int32_t* __restrict__ colT,
                                                                   float* __restrict__ valsT, int32_t rcap, int32_t ecap) {
  extern __shared__ __align__(16) int32_t tc_smem[];
  int32_t* cw_s = tc_smem;                   // [kTcWarps][rcap]: per-warp column counts -> cursors
  int32_t* st_s = cw_s + kTcWarps * rcap;    // [rcap]: column totals -> absolute starts
  int32_t* rp_s = st_s + rcap;               // [rcap]: row pointers relative to z0
  int32_t* cs_s = rp_s + rcap;               // [ecap]: column ids
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  for (int64_t i = blockIdx.x; i < batch; i += gridDim.x) {
    const int64_t g0 = row_off[i], g1 = row_off[i + 1];
    const int32_t n = sizes ? sizes[i] : (int32_t)(g1 - g0);
    const int32_t z0 = row_ptr[g0], z1 = row_ptr[g0 + n], nnz = z1 - z0;
    for (int64_t g = g0 + n + t; g < g1; g += blockDim.x) rowT[g] = z1;  // padding rows: empty
    if (i == batch - 1 && t == 0) rowT[g1] = row_ptr[g1];
    if (n + 1 <= rcap && nnz <= ecap) {
      for (int32_t c = t; c < kTcWarps * rcap; c += blockDim.x) cw_s[c] = 0;
      for (int32_t e = t; e < nnz; e += blockDim.x) cs_s[e] = __ldg(col + z0 + e);
      for (int32_t r = t; r <= n; r += blockDim.x) rp_s[r] = __ldg(row_ptr + g0 + r) - z0;
      __syncthreads();
      const int32_t L = (nnz + kTcWarps - 1) / kTcWarps;
      const int32_t w0 = min(nnz, warp * L), w1 = min(nnz, w0 + L);
      int32_t* cw = cw_s + warp * rcap;
      for (int32_t e0 = w0; e0 < w1; e0 += 32) {  // per-warp column counts
        const int32_t e = e0 + lane;
        const int32_t c = e < w1 ? cs_s[e] : -1 - lane;
        const uint32_t peers = __match_any_sync(0xffffffffu, c);
        if (e < w1 && (peers & lt) == 0) cw[c] += __popc(peers);
        __syncwarp();
      }
      __syncthreads();
      for (int32_t c = t; c < n; c += blockDim.x) {  // per-warp offsets within the column, column totals
        int32_t run = 0;
#pragma unroll
        for (int w = 0; w < kTcWarps; ++w) {
          const int32_t v = cw_s[w * rcap + c];
          cw_s[w * rcap + c] = run;
          run += v;
        }
        st_s[c] = run;
      }
      __syncthreads();
      if (warp == 0) {  // exclusive scan of the totals -> absolute A^T row pointers
        int32_t carry = z0;
        for (int32_t c0 = 0; c0 < n; c0 += 32) {
          const int32_t c = c0 + lane;
          const int32_t v = c < n ? st_s[c] : 0;
          int32_t x = v;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
          }
          if (c < n) {
            st_s[c] = carry + x - v;
            rowT[g0 + c] = carry + x - v;
          }
          carry += __shfl_sync(0xffffffffu, x, 31);
        }
      }
      __syncthreads();
      for (int32_t e0 = w0; e0 < w1; e0 += 32) {  // stable scatter of this warp's range
        const int32_t e = e0 + lane;
        const bool in = e < w1;
        const int32_t c = in ? cs_s[e] : -1 - lane;
        const uint32_t peers = __match_any_sync(0xffffffffu, c);
        if (in) {
          const int32_t slot = st_s[c] + cw[c] + __popc(peers & lt);
          int32_t lo = 0, hi = n - 1;  // source row: the last r with rp[r] <= e (empty rows share rp)
          while (lo < hi) {
            const int32_t mid = (lo + hi + 1) >> 1;
            if (rp_s[mid] <= e) lo = mid;
            else hi = mid - 1;
          }
          BSPMM_CHECK(c >= 0 && c < n && slot >= z0 && slot < z1 && lo >= 0 && lo < n);
          colT[slot] = lo;
          valsT[slot] = __ldg(vals + z0 + e);  // bitwise move
        }
        __syncwarp();
        if (in && (peers & lt) == 0) cw[c] += __popc(peers);
        __syncwarp();
      }
      __syncthreads();  // shared memory reused by the next matrix
      continue;
    }
    // above the capacities: the same counting sort on global memory (counters
    // in rowT's own slots), ranks by a scan of the earlier entries
    for (int32_t c = t; c < n; c += blockDim.x) rowT[g0 + c] = 0;
    __syncthreads();
    for (int32_t e = t; e < nnz; e += blockDim.x) atomicAdd(&rowT[g0 + __ldg(col + z0 + e)], 1);
    __syncthreads();
    if (warp == 0) {
      int32_t carry = z0;
      for (int32_t c0 = 0; c0 < n; c0 += 32) {
        const int32_t c = c0 + lane;
        const int32_t v = c < n ? rowT[g0 + c] : 0;
        int32_t x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int32_t y = __shfl_up_sync(0xffffffffu, x, d);
          if (lane >= d) x += y;
        }
        if (c < n) rowT[g0 + c] = carry + x - v;
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
    }
    __syncthreads();
    for (int32_t e = t; e < nnz; e += blockDim.x) {
      const int32_t c = __ldg(col + z0 + e);
      int32_t rank = 0;
      for (int32_t q = 0; q < e; ++q) rank += __ldg(col + z0 + q) == c ? 1 : 0;
      int32_t lo = 0, hi = n - 1;
      while (lo < hi) {
        const int32_t mid = (lo + hi + 1) >> 1;
        if (__ldg(row_ptr + g0 + mid) - z0 <= e) lo = mid;
        else hi = mid - 1;
      }
      const int32_t slot = rowT[g0 + c] + rank;
      colT[slot] = lo;
      valsT[slot] = __ldg(vals + z0 + e);
    }
    __syncthreads();
  }
}

cudaError_t launch_transpose_csr(int32_t batch, const int64_t* row_off, const int32_t* sizes, const int32_t* row_ptr,
                                 const int32_t* col, const float* vals, int32_t* rowT, int32_t* colT, float* valsT,
                                 int32_t max_rows_hint, int64_t max_nnz_hint, int32_t num_sms, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  if (batch <= 8LL * num_sms && max_rows_hint > 0 && max_nnz_hint > 0) {
    // small (latency-bound) batch: a CTA per matrix (C3 20 -> see DESIGN)
    const int32_t rcap = (max_rows_hint + 1 + 3) & ~3;
    const int32_t ecap = (int32_t)std::min<int64_t>((max_nnz_hint + 3) & ~3LL, 8192);
    const int smem = ((kTcWarps + 2) * rcap + ecap) * 4;
    if (smem <= 96 * 1024) {
      cudaError_t e = cudaSuccess;
      if (smem > 47 * 1024) e = cudaFuncSetAttribute(transpose_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      transpose_cta_kernel<<<batch, kBwdThreads, smem, s>>>(batch, row_off, sizes, row_ptr, col, vals, rowT, colT, valsT,
                                                            rcap, ecap);
      return cudaGetLastError();
    }
  }
  const int64_t need = ((int64_t)batch + kTrWarps - 1) / kTrWarps;
  const int grid = (int)std::min<int64_t>(need, (int64_t)num_sms * 8);
  // row-id capacity: the hinted largest matrix up to 1536 entries (no hint: search)
  const int32_t ridcap = max_nnz_hint > 0 ? (int32_t)std::min<int64_t>((max_nnz_hint + 3) & ~3LL, 1536) : 0;
  // window: 256 columns when the hinted rows fit, else 512 (fewer passes over big matrices)
  const bool small = max_rows_hint > 0 && max_rows_hint <= 256;
  const int smem = kTrWarps * ((small ? 256 : 512) + kTrRp + ridcap) * 4;
  cudaError_t e = cudaSuccess;
  auto go = [&](auto kern) {
    if (smem > 47 * 1024) {  // dynamic + static above the 48 KB default
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return;
    }
    kern<<<grid, kTrWarps * 32, smem, s>>>(batch, row_off, sizes, row_ptr, col, vals, rowT, colT, valsT, ridcap);
    e = cudaGetLastError();
  };
  if (small) go(transpose_csr_kernel<256>);
  else go(transpose_csr_kernel<512>);
  return e;
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
template <int CH, bool STAGED, int PF = 1>
__device__ __forceinline__ void sddmm_rows(int32_t n, int32_t chunks, const float* __restrict__ Bsrc, int64_t bld,
                                           const float* __restrict__ Grow0, int64_t ldg,
                                           const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                           float* __restrict__ out, int lane, int warp, int nw,
                                           uint64_t* bar = nullptr, uint32_t phase = 0) {
  // rows r = warp, warp + nw, ...; the grad_C chunks and row ranges of the
  // next PF rows are in flight while the current row computes (one exposed
  // latency per matrix)
  float4 gq[PF][CH];
  int32_t q0[PF], q1[PF];
  bool ok[CH];
#pragma unroll
  for (int v = 0; v < CH; ++v) ok[v] = lane + 32 * v < chunks;
  auto gload = [&](int32_t r_, float4* dst) {
    const float* grow = Grow0 + (int64_t)r_ * ldg;
#pragma unroll
    for (int v = 0; v < CH; ++v) dst[v] = ok[v] ? ldg_nc_f4(grow + 4 * (lane + 32 * v)) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
#pragma unroll
  for (int f = 0; f < PF; ++f) {
    const int32_t rr = warp + f * nw;
    q0[f] = q1[f] = 0;
    if (rr < n) {
      q0[f] = __ldg(rp + rr);
      q1[f] = __ldg(rp + rr + 1);
      gload(rr, gq[f]);
    }
  }
  // staged: the first rows' grad_C loads are in flight while B_i lands
  if (STAGED) mbar_wait(bar, phase);
  for (int32_t r = warp; r < n; r += nw) {
    const int32_t e0 = q0[0], e1 = q1[0];
    float4 gv[CH];
#pragma unroll
    for (int v = 0; v < CH; ++v) gv[v] = gq[0][v];
#pragma unroll
    for (int f = 0; f + 1 < PF; ++f) {
      q0[f] = q0[f + 1];
      q1[f] = q1[f + 1];
#pragma unroll
      for (int v = 0; v < CH; ++v) gq[f][v] = gq[f + 1][v];
    }
    if (r + PF * nw < n) {
      q0[PF - 1] = __ldg(rp + r + PF * nw);
      q1[PF - 1] = __ldg(rp + r + PF * nw + 1);
      gload(r + PF * nw, gq[PF - 1]);
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
                                                                  const float* __restrict__ G_, int64_t ldg,
                                                                  float* __restrict__ out, int32_t cap_bytes,
                                                                  int32_t dbg) {
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
  // matrix metadata two matrices ahead (loads in flight across an iteration):
  // matrix i's row range is known when its iteration starts, and matrix
  // i + grid's B_i is bulk-prefetched into L2 one matrix ahead, so its TMA
  // copy hits L2 (C5 SDDMM 1099 -> 1074 us; prefetching grad_C_i too measured
  // slower, 1116 us, with ~1 GB of extra DRAM reads: lines evicted before use)
  const int64_t G = gridDim.x;
  auto meta_g = [&](int64_t m) -> int64_t { return m < batch ? row_off[m] : 0; };
  auto meta_n = [&](int64_t m, int64_t g) -> int32_t {
    return m < batch ? (sizes ? sizes[m] : (int32_t)(row_off[m + 1] - g)) : 0;
  };
  int64_t g0 = meta_g(blockIdx.x), g1m = meta_g(blockIdx.x + G);
  int32_t n = meta_n(blockIdx.x, g0), n1m = meta_n(blockIdx.x + G, g1m);
  for (int64_t i = blockIdx.x; i < batch; i += G) {
    const int64_t g2m = meta_g(i + 2 * G);
    const int32_t n2m = meta_n(i + 2 * G, g2m);
    const bool staged = n > 0 && (int64_t)n * k * 4 <= cap_bytes;
    if (threadIdx.x == 0 && n1m > 0 && !(dbg & 512))
      bulk_prefetch_l2(B + g1m * ldb, (uint32_t)(((int64_t)(n1m - 1) * ldb + k) * 4));
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
      sddmm_rows<CH, true>(n, chunks, Bs, k, G_ + g0 * ldg, ldg, row_ptr + g0, col, out, lane, warp, nw, &bar,
                           phase);
      phase ^= 1u;
    } else {
      sddmm_rows<CH, false>(n, chunks, B + g0 * ldb, ldb, G_ + g0 * ldg, ldg, row_ptr + g0, col, out, lane, warp,
                            nw);
    }
    g0 = g1m, n = n1m, g1m = g2m, n1m = n2m;
    __syncthreads();  // every warp is done with Bs before the next matrix's copy
  }
}

// the rare over-capacity matrix of sddmm_struct_kernel, out of line so that
// its registers do not count against the staged loop's
template <int CH>
__device__ __noinline__ void sddmm_rows_global(bool staged, int32_t n, int32_t chunks, const float* Bs, int32_t k,
                                               const float* Bg, int64_t ldb, const float* Gm, int64_t ldg,
                                               const int32_t* rp, const int32_t* col, float* out, uint64_t* bar,
                                               uint32_t phase) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (staged) sddmm_rows<CH, true>(n, chunks, Bs, k, Gm, ldg, rp, col, out, lane, warp, nw, bar, phase);
  else sddmm_rows<CH, false>(n, chunks, Bg, ldb, Gm, ldg, rp, col, out, lane, warp, nw);
}

// Staged SDDMM with the CSR slice in shared memory (round 2, the default for
// streaming batches).  Same CTA shape and B_i staging as sddmm_staged_kernel,
// but no global load sits on a row's chain any more: matrix i + grid's row
// pointers and column ids are cp.async'ed into the other half of a
// double-buffered structure stage while matrix i computes, and so is the
// metadata that addresses them (a 4-slot ring in shared memory: i + grid's
// entry range, i + 3 grid's row range -- no metadata is held in registers
// across the row loop); grad_C rows are prefetched PF rows ahead, and two
// entries share one butterfly (the xor-16 step swaps halves, so lanes 0-15
// reduce entry e and lanes 16-31 entry e + 1 -- every add pairs the same two
// partials as the per-entry butterfly: the same bits).  A matrix whose B_i
// or structure exceeds the stage takes the out-of-line global loop.
struct SdMeta {
  int64_t g;      // first global row
  int64_t gnext;  // row_off[m + 1] (sizes == NULL)
  int32_t n;      // rows (sizes != NULL)
  int32_t ea, eb; // entry range [row_ptr[g], row_ptr[g + n])
  int32_t pad;
};
template <int CH, int PF, bool FULL>
__global__ void __launch_bounds__(kBwdThreads, 3) sddmm_struct_kernel(int32_t batch, int32_t k,
                                                                     const int64_t* __restrict__ row_off,
                                                                     const int32_t* __restrict__ sizes,
                                                                     const int32_t* __restrict__ row_ptr,
                                                                     const int32_t* __restrict__ col,
                                                                     const float* __restrict__ B, int64_t ldb,
                                                                     const float* __restrict__ G_, int64_t ldg,
                                                                     float* __restrict__ out, int32_t cap_bytes,
                                                                     int32_t rcap, int32_t ecap, int32_t dbg) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ SdMeta meta[4];
  float* Bs = reinterpret_cast<float*>(smem);
  int32_t* s_rp = reinterpret_cast<int32_t*>(smem + cap_bytes);  // [2][rcap]
  int32_t* s_col = s_rp + 2 * rcap;                              // [2][ecap]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t G = gridDim.x;
  auto rows_of = [&](const SdMeta& m) -> int32_t { return sizes ? m.n : (int32_t)(m.gnext - m.g); };
  // slot of matrix m: its row range (thread 0) ...
  auto fetch_rows = [&](int64_t m, SdMeta& d) {
    if (m < batch) {
      cp_async8(&d.g, row_off + m);
      if (sizes) cp_async4(&d.n, sizes + m);
      else cp_async8(&d.gnext, row_off + m + 1);
    } else {
      d.g = d.gnext = 0;
      d.n = 0;
    }
  };
  // ... and its entry range (thread 32, once the row range has landed)
  auto fetch_entries = [&](SdMeta& d) {
    const int32_t n = rows_of(d);
    if (n > 0) {
      cp_async4(&d.ea, row_ptr + d.g);
      cp_async4(&d.eb, row_ptr + d.g + n);
    } else {
      d.ea = d.eb = 0;
    }
  };
  auto fits = [&](int32_t n_, int32_t ea, int32_t eb) {
    return n_ > 0 && (int64_t)n_ * k * 4 <= cap_bytes && n_ + 1 <= rcap && eb - ea <= ecap;
  };
  // cp.async a matrix's row pointers and column ids into stage `buf`
  auto stage_struct = [&](int buf, const SdMeta& d) {
    const int32_t n = rows_of(d);
    if (fits(n, d.ea, d.eb)) {
      BSPMM_CHECK(n + 1 <= rcap && d.eb - d.ea <= ecap && d.ea >= 0);
      for (int32_t t = threadIdx.x; t <= n; t += blockDim.x) cp_async4(s_rp + buf * rcap + t, row_ptr + d.g + t);
      for (int32_t t = threadIdx.x; t < d.eb - d.ea; t += blockDim.x) cp_async4(s_col + buf * ecap + t, col + d.ea + t);
    }
  };
  const int64_t i0 = blockIdx.x;
  // prologue: rows of i0 .. i0 + 2G, entries of i0 and i0 + G, i0's structure
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    for (int q = 0; q < 3; ++q) fetch_rows(i0 + q * G, meta[q]);
  }
  cp_async_wait_all();
  __syncthreads();
  if (threadIdx.x == 32)
    for (int q = 0; q < 2; ++q) fetch_entries(meta[q]);
  cp_async_wait_all();
  __syncthreads();
  stage_struct(0, meta[0]);
  cp_async_wait_all();
  __syncthreads();
  uint32_t phase = 0;
  int j = 0;
  for (int64_t i = i0; i < batch; i += G, ++j) {
    const SdMeta& m0 = meta[j & 3];
    const int32_t n0 = rows_of(m0);
    const int64_t g0 = m0.g;
    const int32_t e0a = m0.ea, e0b = m0.eb;
    const bool staged = fits(n0, e0a, e0b);
    if (threadIdx.x == 0) {
      const SdMeta& m1 = meta[(j + 1) & 3];
      const int32_t n1 = rows_of(m1);
      if (n1 > 0 && !(dbg & 512))
        bulk_prefetch_l2(B + m1.g * ldb, (uint32_t)(((int64_t)(n1 - 1) * ldb + k) * 4));
      if (staged) {
        const uint32_t bytes = (uint32_t)n0 * (uint32_t)k * 4u;
        mbar_arrive_expect_tx(&bar, bytes);
        if (ldb == k) {
          bulk_g2s(Bs, B + g0 * ldb, bytes, &bar);
        } else {
          for (int32_t r = 0; r < n0; ++r) bulk_g2s(Bs + (int64_t)r * k, B + (g0 + r) * ldb, (uint32_t)k * 4u, &bar);
        }
      }
      fetch_rows(i + 3 * G, meta[(j + 3) & 3]);
    }
    if (threadIdx.x == 32) fetch_entries(meta[(j + 2) & 3]);
    stage_struct((j + 1) & 1, meta[(j + 1) & 3]);
    if (staged) {
      const int32_t* rp = s_rp + (j & 1) * rcap;
      const int32_t* cs = s_col + (j & 1) * ecap;
      const float* Gm = G_ + g0 * ldg;
      float* o = out + e0a;
      float4 gq[PF][CH];
      auto gload = [&](int32_t r_, float4* dst) {
        const float* grow = Gm + (int64_t)r_ * ldg + 4 * lane;
#pragma unroll
        for (int v = 0; v < CH; ++v)
          dst[v] = (FULL || lane + 32 * v < (k >> 2)) ? ldg_nc_f4(grow + 128 * v) : make_float4(0.f, 0.f, 0.f, 0.f);
      };
#pragma unroll
      for (int f = 0; f < PF; ++f)
        if (warp + f * nw < n0) gload(warp + f * nw, gq[f]);
      mbar_wait(&bar, phase);
      phase ^= 1u;
      for (int32_t r = warp; r < n0; r += nw) {
        float4 gv[CH];
#pragma unroll
        for (int v = 0; v < CH; ++v) gv[v] = gq[0][v];
#pragma unroll
        for (int f = 0; f + 1 < PF; ++f)
#pragma unroll
          for (int v = 0; v < CH; ++v) gq[f][v] = gq[f + 1][v];
        if (r + PF * nw < n0) gload(r + PF * nw, gq[PF - 1]);
        const int32_t ea = rp[r] - e0a, eb = rp[r + 1] - e0a;
        BSPMM_CHECK(0 <= ea && ea <= eb && eb <= e0b - e0a && eb <= ecap && r + 1 < rcap);
        // up to four entries per butterfly: the xor-16 step swaps pairs
        // (lanes < 16 keep entries 0-1, the others 2-3), the xor-8 step
        // swaps within the pair, xor 4, 2, 1 finish; lane 8q writes entry q
        for (int32_t e = ea; e < eb; e += 4) {
          const int32_t m = eb - e;  // warp-uniform
          float p[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            p[q] = 0.f;
            if (q < m) {
              BSPMM_CHECK(cs[e + q] >= 0 && cs[e + q] < n0 && (int64_t)n0 * k * 4 <= cap_bytes);
              const float* bp = Bs + cs[e + q] * k + 4 * lane;
#pragma unroll
              for (int v = 0; v < CH; ++v) {
                if (FULL || lane + 32 * v < (k >> 2)) {
                  const float4 bb = *reinterpret_cast<const float4*>(bp + 128 * v);
                  p[q] = fmaf(gv[v].x, bb.x, p[q]); p[q] = fmaf(gv[v].y, bb.y, p[q]);
                  p[q] = fmaf(gv[v].z, bb.z, p[q]); p[q] = fmaf(gv[v].w, bb.w, p[q]);
                }
              }
            }
          }
          const bool b4 = lane & 16, b3 = lane & 8;
          const float x = __shfl_xor_sync(0xffffffffu, b4 ? p[0] : p[2], 16);
          const float y = __shfl_xor_sync(0xffffffffu, b4 ? p[1] : p[3], 16);
          const float q0 = (b4 ? p[2] : p[0]) + x, q1 = (b4 ? p[3] : p[1]) + y;
          float t = (b3 ? q1 : q0) + __shfl_xor_sync(0xffffffffu, b3 ? q0 : q1, 8);
#pragma unroll
          for (int d = 4; d > 0; d >>= 1) t += __shfl_xor_sync(0xffffffffu, t, d);
          const int32_t q = (b4 ? 2 : 0) + (b3 ? 1 : 0);
          if ((lane & 7) == 0 && q < m) o[e + q] = t;
        }
      }
    } else if (n0 > 0) {  // B_i or the structure above the stage: the global loop
      sddmm_rows_global<CH>(false, n0, k >> 2, Bs, k, B + g0 * ldb, ldb, G_ + g0 * ldg, ldg, row_ptr + g0, col,
                            out, &bar, 0);
    }
    cp_async_wait_all();  // the next matrix's structure and the metadata ring
    __syncthreads();      // ... visible to every warp; every warp is done with Bs
  }
}

// ---------------------------------------------------------------------------
// Fused backward for streaming batches (both adjoints, round 2): per matrix,
// grad_C_i is staged in shared memory ONCE and feeds both
//   grad_B_i = A_i^T grad_C_i      (bitwise the storage-order fp32 sum over
//                                   the canonical A_i^T, as the transpose +
//                                   forward-kernel path computes it)
//   grad_vals_e = <grad_C[row_e], B[col_e]>   (the SDDMM's bits)
// so grad_C is read once and no A^T is written to or read from HBM: C5 moves
// B + grad_C in and grad_B out (8.1 GB) instead of the separate kernels'
// 10.9 GB plus the transpose pass.  CTA flow per matrix (3 CTAs x 8 warps per
// SM, persistent): the next matrix's CSR slice (row pointers, column ids,
// values) is cp.async'ed into the other half of a double-buffered stage, its
// metadata through the SDDMM kernel's 4-slot ring; grad_C_i lands by one
// bulk copy while warp 0 transposes A_i in shared memory (column counts by
// shared atomics, a warp scan, then a scatter 32 entries at a time in storage
// order with equal columns ranked by __match_any_sync -- a stable counting
// sort, so A^T comes out in canonical (row, col, original position) order);
// then warp
// w owns rows c = w, w + 8, ... of A^T (= rows of B and grad_B): B's row in
// registers (loaded one row ahead), every entry (r, v, e) of the row reads
// grad_C's row r from shared memory once for the FMA into grad_B and the dot
// product with B's row (two entries per butterfly, the xor-16 step swapping
// them).  A matrix above the stage capacities takes the out-of-line global
// path (below).
template <int CH>
__device__ __noinline__ void bwd_fused_global(int32_t n, int32_t k, int64_t g0, const int32_t* __restrict__ row_ptr,
                                              const int32_t* __restrict__ col, const float* __restrict__ vals,
                                              const float* __restrict__ B, int64_t ldb,
                                              const float* __restrict__ Gg, int64_t ldg, float* __restrict__ gB,
                                              int64_t ldgb, float* __restrict__ gvals) {
  // over-capacity matrix: grad_vals by the SDDMM's global loop; grad_B row c
  // by scanning the matrix's entries in storage order for column c (the
  // canonical A^T order), grad_C rows from global memory
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  sddmm_rows<CH, false>(n, k >> 2, B + g0 * ldb, ldb, Gg + g0 * ldg, ldg, row_ptr + g0, col, gvals, lane, warp, nw);
  const int32_t z0 = __ldg(row_ptr + g0), z1 = __ldg(row_ptr + g0 + n);
  for (int32_t c = warp; c < n; c += nw) {
    for (int32_t j = lane; j < k; j += 32) {
      float acc = 0.f;
      int32_t r = 0;
      for (int32_t e = z0; e < z1; ++e) {
        while (e >= __ldg(row_ptr + g0 + r + 1)) ++r;
        if (__ldg(col + e) == c) acc = fmaf(__ldg(vals + e), __ldg(Gg + (g0 + r) * ldg + j), acc);
      }
      gB[(g0 + c) * ldgb + j] = acc;
    }
  }
}

template <int CH, bool FULL>
__global__ void __launch_bounds__(kBwdThreads, 3) backward_fused_kernel(
    int32_t batch, int32_t k, const int64_t* __restrict__ row_off, const int32_t* __restrict__ sizes,
    const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col, const float* __restrict__ vals,
    const float* __restrict__ B, int64_t ldb, const float* __restrict__ G_, int64_t ldg, float* __restrict__ gB,
    int64_t ldgb, float* __restrict__ gvals, int32_t cap_bytes, int32_t rcap, int32_t ecap, int32_t dbg) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ SdMeta meta[4];
  float* Gs = reinterpret_cast<float*>(smem);
  int32_t* s_rp = reinterpret_cast<int32_t*>(smem + cap_bytes);  // [2][rcap]
  int32_t* s_col = s_rp + 2 * rcap;                              // [2][ecap]
  float* s_val = reinterpret_cast<float*>(s_col + 2 * ecap);     // [2][ecap]
  int32_t* t_rp2 = reinterpret_cast<int32_t*>(s_val + 2 * ecap);  // [2][rcap]: A^T row pointers (column counts
                                                                  // first), double-buffered: the next matrix's
                                                                  // counters are zeroed while this one runs
  int32_t* t_row = t_rp2 + 2 * rcap;                             // [ecap]: A^T entry -> source row
  float* t_val = reinterpret_cast<float*>(t_row + ecap);         // [ecap]
  int32_t* t_pos = reinterpret_cast<int32_t*>(t_val + ecap);     // [ecap]: A^T entry -> A's entry (local)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t G = gridDim.x;
  auto rows_of = [&](const SdMeta& m) -> int32_t { return sizes ? m.n : (int32_t)(m.gnext - m.g); };
  auto fetch_rows = [&](int64_t m, SdMeta& d) {
    if (m < batch) {
      cp_async8(&d.g, row_off + m);
      if (sizes) cp_async4(&d.n, sizes + m);
      else cp_async8(&d.gnext, row_off + m + 1);
    } else {
      d.g = d.gnext = 0;
      d.n = 0;
    }
  };
  auto fetch_entries = [&](SdMeta& d) {
    const int32_t n = rows_of(d);
    if (n > 0) {
      cp_async4(&d.ea, row_ptr + d.g);
      cp_async4(&d.eb, row_ptr + d.g + n);
    } else {
      d.ea = d.eb = 0;
    }
  };
  auto fits = [&](int32_t n_, int32_t ea, int32_t eb) {
    return n_ > 0 && (int64_t)n_ * k * 4 <= cap_bytes && n_ + 1 <= rcap && eb - ea <= ecap;
  };
  auto stage_struct = [&](int buf, const SdMeta& d) {
    const int32_t n = rows_of(d);
    if (fits(n, d.ea, d.eb)) {
      BSPMM_CHECK(n + 1 <= rcap && d.eb - d.ea <= ecap && d.ea >= 0);
      for (int32_t t = threadIdx.x; t <= n; t += blockDim.x) cp_async4(s_rp + buf * rcap + t, row_ptr + d.g + t);
      for (int32_t t = threadIdx.x; t < d.eb - d.ea; t += blockDim.x) {
        cp_async4(s_col + buf * ecap + t, col + d.ea + t);
        cp_async4(s_val + buf * ecap + t, vals + d.ea + t);
      }
    }
  };
  const int64_t i0 = blockIdx.x;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    for (int q = 0; q < 3; ++q) fetch_rows(i0 + q * G, meta[q]);
  }
  cp_async_wait_all();
  __syncthreads();
  if (threadIdx.x == 32)
    for (int q = 0; q < 2; ++q) fetch_entries(meta[q]);
  cp_async_wait_all();
  __syncthreads();
  stage_struct(0, meta[0]);
  for (int32_t c = threadIdx.x; c < 2 * rcap; c += blockDim.x) t_rp2[c] = 0;  // column counters
  cp_async_wait_all();
  __syncthreads();
  uint32_t phase = 0;
  int j = 0;
  for (int64_t i = i0; i < batch; i += G, ++j) {
    const SdMeta& m0 = meta[j & 3];
    const int32_t n0 = rows_of(m0);
    const int64_t g0 = m0.g;
    const int32_t e0a = m0.ea, nnz = m0.eb - m0.ea;
    const bool staged = fits(n0, m0.ea, m0.eb);
    int32_t* t_rp = t_rp2 + (j & 1) * rcap;
    // (no L2 prefetch of the next matrix's grad_C / B rows: with the grad_B
    // stores streaming through L2 the prefetched lines were evicted before
    // use -- DRAM reads 8.27 GB instead of 5.44, 1669 vs 1388 us on C5;
    // grad_C alone 1418 us)
    if (threadIdx.x == 0) {
      if (staged) {
        const uint32_t bytes = (uint32_t)n0 * (uint32_t)k * 4u;
        mbar_arrive_expect_tx(&bar, bytes);
        if (ldg == k) {
          bulk_g2s(Gs, G_ + g0 * ldg, bytes, &bar);
        } else {
          for (int32_t r = 0; r < n0; ++r) bulk_g2s(Gs + (int64_t)r * k, G_ + (g0 + r) * ldg, (uint32_t)k * 4u, &bar);
        }
      }
      fetch_rows(i + 3 * G, meta[(j + 3) & 3]);
    }
    if (threadIdx.x == 32) fetch_entries(meta[(j + 2) & 3]);
    stage_struct((j + 1) & 1, meta[(j + 1) & 3]);
    {  // the next matrix's column counters (that buffer was last read a matrix ago)
      int32_t* t_nx = t_rp2 + ((j + 1) & 1) * rcap;
      for (int32_t c = threadIdx.x; c < rcap; c += blockDim.x) t_nx[c] = 0;
    }
    if (staged) {
      const int32_t* rp = s_rp + (j & 1) * rcap;
      const int32_t* cs = s_col + (j & 1) * ecap;
      const float* vs = s_val + (j & 1) * ecap;
      // B's first row of this warp (registers), in flight during the transpose
      float4 bq[CH];
      auto bload = [&](int32_t c_, float4* dst) {
        const float* brow = B + (g0 + c_) * ldb + 4 * lane;
#pragma unroll
        for (int v = 0; v < CH; ++v)
          dst[v] = (FULL || lane + 32 * v < (k >> 2)) ? ldg_nc_f4(brow + 128 * v) : make_float4(0.f, 0.f, 0.f, 0.f);
      };
      if (warp < n0) bload(warp, bq);
      // ---- A_i^T in shared memory (while grad_C_i lands): column counts by
      // shared atomics (the counters were zeroed at the end of the previous
      // matrix), a warp scan, then every entry's slot = its column's start +
      // the number of earlier entries of that column (stable)
      for (int32_t e = threadIdx.x; e < nnz; e += blockDim.x) {
        BSPMM_CHECK(cs[e] >= 0 && cs[e] < n0 && n0 < rcap);
        atomicAdd(&t_rp[cs[e] + 1], 1);
      }
      __syncthreads();
      if (warp == 0) {  // inclusive scan of t_rp[1..n0] -> row pointers of A^T (t_rp[0] = 0)
        int32_t carry = 0;
        for (int32_t c0 = 1; c0 <= n0; c0 += 32) {
          const int32_t c = c0 + lane;
          int32_t x = c <= n0 ? t_rp[c] : 0;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
          }
          if (c <= n0) t_rp[c] = carry + x;
          carry += __shfl_sync(0xffffffffu, x, 31);
        }
      }
      __syncthreads();
      for (int32_t e = threadIdx.x; e < nnz; e += blockDim.x) {
        const int32_t c = cs[e];
        int32_t rank = 0, q = 0;
        for (; q + 4 <= e; q += 4) {  // 4 column ids per shared load (the stage is 16-byte aligned)
          const int4 c4 = *reinterpret_cast<const int4*>(cs + q);
          rank += (c4.x == c) + (c4.y == c) + (c4.z == c) + (c4.w == c);
        }
        for (; q < e; ++q) rank += cs[q] == c ? 1 : 0;
        int32_t lo = 0, hi = n0 - 1;  // source row: the last r with rp[r] - e0a <= e
        while (lo < hi) {
          const int32_t mid = (lo + hi + 1) >> 1;
          if (rp[mid] - e0a <= e) lo = mid;
          else hi = mid - 1;
        }
        const int32_t slot = t_rp[c] + rank;
        BSPMM_CHECK(slot >= t_rp[c] && slot < t_rp[c + 1] && slot < nnz && lo >= 0 && lo < n0);
        t_row[slot] = lo;
        t_val[slot] = vs[e];
        t_pos[slot] = e;
      }
      __syncthreads();
      mbar_wait(&bar, phase);
      phase ^= 1u;
      float* ov = gvals + e0a;
      for (int32_t c = warp; c < n0; c += nw) {
        float4 b[CH];
#pragma unroll
        for (int v = 0; v < CH; ++v) b[v] = bq[v];
        if (c + nw < n0) bload(c + nw, bq);
        float4 acc[CH];
#pragma unroll
        for (int v = 0; v < CH; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        const int32_t sa = t_rp[c], sb = t_rp[c + 1];
        BSPMM_CHECK(0 <= sa && sa <= sb && sb <= nnz);
        for (int32_t s2 = sa; s2 < sb; s2 += 2) {
          const bool two = s2 + 1 < sb;  // warp-uniform
          BSPMM_CHECK(t_row[s2] >= 0 && t_row[s2] < n0 && t_pos[s2] >= 0 && t_pos[s2] < nnz);
          const float* g0p = Gs + t_row[s2] * k + 4 * lane;
          const float* g1p = Gs + t_row[two ? s2 + 1 : s2] * k + 4 * lane;
          const float v0 = t_val[s2], v1 = two ? t_val[s2 + 1] : 0.f;
          float p0 = 0.f, p1 = 0.f;
#pragma unroll
          for (int v = 0; v < CH; ++v) {
            if (FULL || lane + 32 * v < (k >> 2)) {
              const float4 ga = *reinterpret_cast<const float4*>(g0p + 128 * v);
              acc[v].x = fmaf(v0, ga.x, acc[v].x); acc[v].y = fmaf(v0, ga.y, acc[v].y);
              acc[v].z = fmaf(v0, ga.z, acc[v].z); acc[v].w = fmaf(v0, ga.w, acc[v].w);
              p0 = fmaf(ga.x, b[v].x, p0); p0 = fmaf(ga.y, b[v].y, p0);
              p0 = fmaf(ga.z, b[v].z, p0); p0 = fmaf(ga.w, b[v].w, p0);
              if (two) {
                const float4 gb = *reinterpret_cast<const float4*>(g1p + 128 * v);
                acc[v].x = fmaf(v1, gb.x, acc[v].x); acc[v].y = fmaf(v1, gb.y, acc[v].y);
                acc[v].z = fmaf(v1, gb.z, acc[v].z); acc[v].w = fmaf(v1, gb.w, acc[v].w);
                p1 = fmaf(gb.x, b[v].x, p1); p1 = fmaf(gb.y, b[v].y, p1);
                p1 = fmaf(gb.z, b[v].z, p1); p1 = fmaf(gb.w, b[v].w, p1);
              }
            }
          }
          // xor-16 step with the pair swapped (lanes < 16: entry s2, others s2 + 1)
          const bool hi16 = lane & 16;
          float pp = (hi16 ? p1 : p0) + __shfl_xor_sync(0xffffffffu, hi16 ? p0 : p1, 16);
#pragma unroll
          for (int d = 8; d > 0; d >>= 1) pp += __shfl_xor_sync(0xffffffffu, pp, d);
          if (lane == 0) ov[t_pos[s2]] = pp;
          if (lane == 16 && two) ov[t_pos[s2 + 1]] = pp;
        }
        float* grow = gB + (g0 + c) * ldgb + 4 * lane;
#pragma unroll
        for (int v = 0; v < CH; ++v)
          if (FULL || lane + 32 * v < (k >> 2)) stg_cs_f4(grow + 128 * v, acc[v]);
      }
    } else if (n0 > 0) {
      bwd_fused_global<CH>(n0, k, g0, row_ptr, col, vals, B, ldb, G_, ldg, gB, ldgb, gvals);
    }
    cp_async_wait_all();  // the next matrix's structure and the metadata ring
    __syncthreads();      // ... visible to every warp; every warp is done with Gs and the A^T stage
  }
}

cudaError_t launch_backward_fused(int32_t batch, int32_t k, const int64_t* row_off, const int32_t* sizes,
                                  const int32_t* row_ptr, const int32_t* col, const float* vals, const float* B,
                                  int64_t ldb, const float* G, int64_t ldg, float* gB, int64_t ldgb, float* gvals,
                                  int32_t max_rows_hint, int64_t max_nnz_hint, int32_t num_sms, int32_t dbg,
                                  cudaStream_t s, bool* used) {
  *used = false;
  const int chunks = k >> 2;
  const bool vec = (k % 4 == 0) && (ldb % 4 == 0) && (ldg % 4 == 0) && (ldgb % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(G) |
                     reinterpret_cast<uintptr_t>(gB)) & 15u) == 0;
  // streaming batches with hints that bound every matrix (the stage is sized
  // from them); k <= 256 (two float4 per lane)
  if (!vec || !vals || k > 256 || max_rows_hint <= 0 || max_nnz_hint <= 0 || max_nnz_hint > 1024 ||
      batch <= 8LL * num_sms)
    return cudaSuccess;
  const int32_t cap = (int32_t)(((int64_t)max_rows_hint * k * 4 + 127) & ~127LL);
  // multiples of 4 entries: the column-id stage is read 16 bytes at a time
  const int32_t rcap = (max_rows_hint + 1 + 3) & ~3, ecap = (int32_t)((max_nnz_hint + 3) & ~3LL);
  const int32_t sbytes = cap + 2 * (rcap + 2 * ecap) * 4 + (2 * rcap + 3 * ecap) * 4;
  if (sbytes > 74 * 1024) return cudaSuccess;  // 3 CTAs per SM
  cudaError_t e = cudaSuccess;
  auto go = [&](auto kern) {
    if (sbytes > 47 * 1024) {  // dynamic + static above the 48 KB default
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sbytes);
      if (e != cudaSuccess) return;
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBwdThreads, sbytes);
    if (e != cudaSuccess) return;
    const int grid = (int)std::min<int64_t>(batch, (int64_t)num_sms * std::max(per_sm, 1));
    kern<<<grid, kBwdThreads, sbytes, s>>>(batch, k, row_off, sizes, row_ptr, col, vals, B, ldb, G, ldg, gB, ldgb,
                                           gvals, cap, rcap, ecap, dbg);
    e = cudaGetLastError();
    *used = e == cudaSuccess;
  };
  if (chunks == 64) go(backward_fused_kernel<2, true>);
  else if (chunks == 32) go(backward_fused_kernel<1, true>);
  else if (chunks <= 32) go(backward_fused_kernel<1, false>);
  else go(backward_fused_kernel<2, false>);
  return e;
}

cudaError_t launch_sddmm(int32_t batch, int32_t k, const int64_t* row_off, const int32_t* sizes,
                         const int32_t* row_ptr, const int32_t* col, const float* B, int64_t ldb, const float* G,
                         int64_t ldg, float* out, int32_t max_rows_hint, int64_t max_nnz_hint, int32_t num_sms,
                         int32_t dbg, cudaStream_t s) {
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
      if (cap > 47 * 1024) {  // dynamic + static above the 48 KB default
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
        if (e != cudaSuccess) return;
      }
      kern<<<grid, kBwdThreads, cap, s>>>(batch, k, row_off, sizes, row_ptr, col, B, ldb, G, ldg, out, cap, dbg);
      e = cudaGetLastError();
    };
    if ((dbg & kDbgSddmmGlobalStruct) || ch > 2) {  // structure read from global memory (k > 256: the
                                                    // struct kernel would spill at 3 CTAs per SM)
      if (ch <= 1) go(sddmm_staged_kernel<1>);
      else if (ch <= 2) go(sddmm_staged_kernel<2>);
      else go(sddmm_staged_kernel<4>);
      return e;
    }
    // structure stage: two buffers of (hinted rows + 1) row pointers and
    // (hinted entries) column ids; matrices above it take the global loop
    const int32_t rcap = (max_rows_hint > 0 ? std::min<int32_t>(max_rows_hint, 1024) : 256) + 1;
    const int32_t ecap = max_nnz_hint > 0 ? (int32_t)std::min<int64_t>(max_nnz_hint, 4096) : 2048;
    const int32_t sbytes = cap + 2 * (rcap + ecap) * 4;
    auto go2 = [&](auto kern) {
      if (sbytes > 47 * 1024) {  // dynamic + static above the 48 KB default
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sbytes);
        if (e != cudaSuccess) return;
      }
      // persistent: exactly the resident CTAs (a partial last wave of a
      // larger grid idles a third of the SMs at the end)
      int per_sm = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBwdThreads, sbytes);
      if (e != cudaSuccess) return;
      const int grid2 = (int)std::min<int64_t>(batch, (int64_t)num_sms * std::max(per_sm, 1));
      kern<<<grid2, kBwdThreads, sbytes, s>>>(batch, k, row_off, sizes, row_ptr, col, B, ldb, G, ldg, out, cap, rcap,
                                              ecap, dbg);
      e = cudaGetLastError();
    };
    const bool pf2 = (dbg & kDbgSddmmPf2) != 0;
    if (chunks == 64) pf2 ? go2(sddmm_struct_kernel<2, 2, true>) : go2(sddmm_struct_kernel<2, 1, true>);
    else if (chunks == 32) go2(sddmm_struct_kernel<1, 1, true>);
    else if (ch <= 1) go2(sddmm_struct_kernel<1, 1, false>);
    else go2(sddmm_struct_kernel<2, 1, false>);
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
