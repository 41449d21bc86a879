// offsets.cu — batch-offset builder (hot-path row a-1) and the BSPMM_VALIDATE
// index checks.
//
// The paper builds the list of per-matrix pointers on the host and copies it
// host->device inside the timed region; at small n_B
// that copy decides the race against cuBLAS (:359).  Here the offsets are an
// int64 exclusive scan of the int32 sizes computed on the device in one
// launch: a single-pass decoupled look-back scan.  Each CTA takes a tile of
// 4096 sizes (ticket order, so predecessors are always running), loads it
// coalesced and transposes through shared memory, block-scans, publishes its
// aggregate, looks back over its predecessors' aggregates / inclusive prefixes
// (epoch-tagged status words: no per-call memset) and writes its offsets back
// coalesced.
#include <cstdint>

#include "internal.h"

namespace bspmm {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(kScanThreads) offsets_kernel(int32_t batch, const int32_t* __restrict__ sizes,
                                                               int64_t* __restrict__ out, ScanState st) {
  // s_in (int32, padded every 32) and s_out (int64, padded every 16) share one buffer:
  // s_in is fully consumed into registers before the barrier that precedes s_out's writes
  __shared__ int64_t s_out[kScanTile + kScanTile / 16];
  int32_t* s_in = reinterpret_cast<int32_t*>(s_out);
  __shared__ int64_t warp_tot[kScanThreads / 32];
  __shared__ int64_t s_excl;
  __shared__ int32_t s_tile;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  // let a PDL-launched dependent (the SpMM) start its prologue now
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (t == 0) {
    // ticket order guarantees every predecessor tile is already running; the
    // CTA drawing the last ticket resets the counter for the next launch
    const unsigned long long tk = atomicAdd(st.ticket, 1ULL);
    if (tk == (unsigned long long)gridDim.x - 1) atomicExch(st.ticket, 0ULL);
    s_tile = (int32_t)tk;
  }
  __syncthreads();
  const int32_t tile = s_tile;
  const int64_t base = (int64_t)tile * kScanTile;
  // coalesced load, transpose to thread-contiguous through padded smem
#pragma unroll
  for (int it = 0; it < kScanItems; ++it) {
    const int p = it * kScanThreads + t;
    const int64_t g = base + p;
    s_in[p + (p >> 5)] = g < batch ? __ldg(sizes + g) : 0;
  }
  __syncthreads();
  int32_t v[kScanItems];
  int64_t sum = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int p = t * kScanItems + j;
    v[j] = s_in[p + (p >> 5)];
    sum += v[j];
  }
  // block exclusive scan of the thread sums
  int64_t x = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  int64_t wpre = 0, total = 0;
#pragma unroll
  for (int q = 0; q < kScanThreads / 32; ++q) {
    if (q < w) wpre += warp_tot[q];
    total += warp_tot[q];
  }
  const int64_t thread_excl = wpre + x - sum;
  // decoupled look-back, warp-parallel: lane l inspects predecessor tile - 1 - l
  if (w == 0) {
    const uint32_t tag = st.epoch << 2;
    int64_t excl = 0;
    if (tile == 0) {
      if (lane == 0) {
        st.incl[0] = total;
        __threadfence();
        st_volatile_u32(st.flags, tag | 2u);
      }
    } else {
      if (lane == 0) {
        st.agg[tile] = total;
        __threadfence();
        st_volatile_u32(st.flags + tile, tag | 1u);
      }
      for (int32_t hi = tile - 1; hi >= 0; hi -= 32) {
        const int32_t p = hi - lane;
        uint32_t state = 2u;  // tiles before 0 act as an inclusive zero
        int64_t val = 0;
        if (p >= 0) {
          uint32_t f;
          do {
            f = ld_volatile_u32(st.flags + p);
          } while ((f & ~3u) != tag || (f & 3u) == 0u);
          __threadfence();
          state = f & 3u;
          val = state == 2u ? *((volatile int64_t*)(st.incl + p)) : *((volatile int64_t*)(st.agg + p));
        }
        const uint32_t incl_mask = __ballot_sync(0xffffffffu, state == 2u);
        const int stop = incl_mask ? __ffs(incl_mask) - 1 : 31;  // nearest inclusive predecessor
        int64_t part = lane <= stop ? val : 0;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(0xffffffffu, part, d);
        excl += part;
        if (incl_mask) break;
      }
      if (lane == 0) {
        st.incl[tile] = excl + total;
        __threadfence();
        st_volatile_u32(st.flags + tile, tag | 2u);
      }
    }
    if (lane == 0) s_excl = excl;
  }
  __syncthreads();
  int64_t run = s_excl + thread_excl;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    run += v[j];
    const int p = t * kScanItems + j;
    s_out[p + (p >> 4)] = run;
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kScanItems; ++it) {
    const int p = it * kScanThreads + t;
    const int64_t g = base + p;
    if (g < batch) out[g + 1] = s_out[p + (p >> 4)];
  }
  if (tile == 0 && t == 0) out[0] = 0;
}

int32_t scan_tiles(int32_t batch) { return (int32_t)ceil_div(batch, kScanTile); }

cudaError_t launch_offsets(int32_t batch, const int32_t* sizes, int64_t* out, const ScanState& st,
                           cudaStream_t s) {
  if (batch <= 0) return cudaMemsetAsync(out, 0, sizeof(int64_t), s);
  offsets_kernel<<<scan_tiles(batch), kScanThreads, 0, s>>>(batch, sizes, out, st);
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
