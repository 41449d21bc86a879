// spmm_tile.cu — the batched CSR SpMM for small batches (hot-path rows a-4,
// a-5, a-6 for the latency-bound configs, BASELINE.json configs 1-4): one
// short-lived CTA per TILE = (matrix i, block of cb float4 columns).
//
// What it computes is exactly spmm_csr.cu's operation (PAPER.md Fig.
// algo:code_swa_spmm_csr, lines 196-207, batched as in §IV-C): for every
// matrix i, row r < n_i and column c < k
//     C[g][c] = sum_{e in row g} vals[e] * B[row_off[i] + col[e]][c],
// g = row_off[i] + r, fp32 FMA in CSR storage order from +0 (bitwise O3').
//
// Why a second kernel.  A batch of 100 graphs is 100 units of work for 148
// SMs; the persistent pipeline of spmm_csr.cu stages each B_i whole in one
// CTA, so a third of the SMs idle and every CTA serialises landing (100 KB
// per SM on config 4) and its row pass.  Here the paper's column cache
// blocking (p column blocks per SpMM) is used
// to cut the batch into MANY small independent tiles instead: B_i[:, block]
// and C_i[:, block] depend on nothing else (a C column needs only the same B
// column), so a tile is a complete little SpMM.  With cb chosen so that the
// batch makes ~8-16 tiles per SM, every SM holds many CTAs at once and they
// overlap: one tile's loads land while another computes and a third stores --
// the same overlap a plain copy kernel gets, with no producer/consumer
// barrier spanning a whole SM.
//
// Per CTA (128 threads, several per SM):
//   RT1  the matrix's row offset and size (fused offsets: a block sum of the
//        sizes before it when row_off == NULL);
//   B    the tile B_i[:, c0 .. c0+cw) (n_i x cw float4) into shared memory by
//        16-byte cp.async, issued at once;
//   RT2  the matrix's row pointers (and its first/last entry), RT3 its (col,
//        val) run -> shared memory, while B lands;
//   row pass: thread (row slot, column) -- cb lanes per row, the paper's
//        subWarp lanes on lane-strided columns in
//        float4 chunks -- storage-order FMA over the row's entries, one
//        128-bit streaming store per (row, chunk); empty rows store +0.
// A matrix whose tile or structure does not fit the planned capacity reads
// them from global memory instead (the paper's case 3),
// decided per CTA: correct for any size, fast for the planned ones.
#include <algorithm>
#include <cstdint>

#include "internal.h"
#include "ptx.cuh"

namespace bspmm {

constexpr int kTileThreads = 128;

struct TileParams {
  int32_t batch, k4, tiles;
  int32_t cap_rows, cap_nnz;           // staging capacity: rows of a tile, entries of a matrix
  int32_t rp_off, col_off, val_off;    // shared-memory carve-up (bytes) after the B tile
  const int64_t* __restrict__ row_off;
  const int32_t* __restrict__ sizes;
  const int32_t* __restrict__ row_ptr;
  const int32_t* __restrict__ col;
  const float* __restrict__ vals;
  const float4* __restrict__ B;
  int64_t ldb4;
  float4* __restrict__ C;
  int64_t ldc4;
  const float4* __restrict__ bias;  // GCN epilogue (EPI 1): C += rowsum(A) (x) bias
  int32_t accumulate;               // GCN epilogue: C += previous C
  int32_t tma;                      // 1: B tile by 2-D tensor TMA (maps: box {4 CB, 2^b rows})
  int32_t rp_first;                 // 1: the row-pointer round trip is issued before the B tile
  int32_t dbg_bits;                 // 1: no TMA descriptor prefetch
  unsigned long long* trace;        // debug: per-CTA phase timestamps (globaltimer ns), or null
  // SparseTensor input (spmm_tile_coo_kernel): per-matrix entry offsets, local
  // (row, col) pairs, values; scratch for the conversion after val_off
  const int64_t* __restrict__ nnz_off;
  const int32_t* __restrict__ idx;
  int32_t pair_off, cval_off, slot_off, cnt_off;
  int* err;                         // bit 64: a matrix beyond the hinted capacity (skipped)
  uint64_t b_lo, b_hi;              // B's allocation (0: no pre-wait prefetch)
  uint64_t s_lo[3], s_hi[3];        // structure allocations (CSR row_ptr, col, vals; COO -, idx, vals)
};

// Pre-wait prologue (programmatic dependent launch): CTA b < batch prefetches
// matrix b's B rows into L2 BEFORE griddepcontrol.wait, while the previous
// kernel drains -- in a stream of launches, a launch's B reads overlap the
// previous launch's tail and stores.  The row range is read with a relaxed
// load that may race with the previous kernel (if it writes row_off); the
// prefetch is only a hint, clipped to B's allocation, and every value the
// kernel uses is read again after the wait.
__device__ __forceinline__ void tile_prefetch_b(const TileParams& p) {
  // thread 0: B rows; thread 32 (another warp, so that its second dependent
  // read does not hold up warp 0 after the wait): the structure
  if (!p.b_hi || !p.row_off || (threadIdx.x & ~32u) != 0 || blockIdx.x >= (unsigned)p.batch) return;
  const int64_t i = blockIdx.x;
  const int64_t g0 = ld_relaxed_s64(p.row_off + i);
  const int64_t g1 = p.sizes ? g0 + ld_relaxed_s32(p.sizes + i) : ld_relaxed_s64(p.row_off + i + 1);
  if (g1 <= g0 || g1 - g0 > (1 << 20)) return;
  BSPMM_CHECK(p.b_lo < p.b_hi);
  if (threadIdx.x == 0) {
    prefetch_l2_clipped(reinterpret_cast<uint64_t>(p.B + g0 * p.ldb4), (uint64_t)(g1 - g0) * p.ldb4 * 16, p.b_lo,
                        p.b_hi);
    return;
  }
  // ... and its structure: the row-pointer slice and the (col, val) run (CSR),
  // or the SparseTensor slice (COO)
  int64_t z0, z1;
  if (p.nnz_off) {
    if (!p.s_hi[1]) return;
    z0 = ld_relaxed_s64(p.nnz_off + i);
    z1 = ld_relaxed_s64(p.nnz_off + i + 1);
    if (z1 <= z0 || z1 - z0 > (1 << 24)) return;
    prefetch_l2_clipped(reinterpret_cast<uint64_t>(p.idx + 2 * z0), (uint64_t)(z1 - z0) * 8, p.s_lo[1], p.s_hi[1]);
  } else {
    if (!p.s_hi[0]) return;
    prefetch_l2_clipped(reinterpret_cast<uint64_t>(p.row_ptr + g0), (uint64_t)(g1 - g0 + 1) * 4, p.s_lo[0],
                        p.s_hi[0]);
    const uint64_t rp = reinterpret_cast<uint64_t>(p.row_ptr);
    if (rp + 4 * (uint64_t)g0 < p.s_lo[0] || rp + 4 * (uint64_t)g1 + 4 > p.s_hi[0]) return;
    // and the (col, val) run (a second dependent read): with cp.async staging
    // it measured slower on C4 (6.1 vs 5.85 us), with TMA staging -- the
    // default -- C4 5.52-5.60 vs 5.60-5.62 and C2 2.87 vs 3.04 us; debug bit
    // 26 leaves it out
    if (p.dbg_bits & 2) return;
    z0 = ld_relaxed_s32(p.row_ptr + g0);
    z1 = ld_relaxed_s32(p.row_ptr + g1);
    if (z1 <= z0 || z1 - z0 > (1 << 24) || !p.s_hi[1]) return;
    prefetch_l2_clipped(reinterpret_cast<uint64_t>(p.col + z0), (uint64_t)(z1 - z0) * 4, p.s_lo[1], p.s_hi[1]);
  }
  prefetch_l2_clipped(reinterpret_cast<uint64_t>(p.vals + z0), (uint64_t)(z1 - z0) * 4, p.s_lo[2], p.s_hi[2]);
}

__device__ __forceinline__ void tile_trace(const TileParams& p, int slot) {
  if (p.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    p.trace[(size_t)blockIdx.x * 32 + slot] = t;
  }
}

// sum of sizes[0 .. i) over the CTA (fused offsets builder, packed layout):
// every load of a thread in flight before any add (one round trip)
__device__ __forceinline__ int64_t tile_sizes_prefix(const int32_t* __restrict__ sizes, int32_t i) {
  __shared__ int64_t part[kTileThreads / 32];
  int64_t s = 0;
  for (int32_t m0 = 0; m0 < i; m0 += 8 * kTileThreads) {
    int32_t v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int32_t m = m0 + threadIdx.x + q * kTileThreads;
      v[q] = m < i ? __ldg(sizes + m) : 0;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) s += v[q];
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  int64_t tot = 0;
#pragma unroll
  for (int w = 0; w < kTileThreads / 32; ++w) tot += part[w];
  return tot;
}

__device__ __forceinline__ void fma4(float4& acc, float a, const float4& b) {
  acc.x = fmaf(a, b.x, acc.x);
  acc.y = fmaf(a, b.y, acc.y);
  acc.z = fmaf(a, b.z, acc.z);
  acc.w = fmaf(a, b.w, acc.w);
}

template <int EPI>
__device__ __forceinline__ void tile_store(const TileParams& p, float4* dst, int32_t colf4, float4 acc, float rs) {
  if (EPI == 1) {
    if (p.bias) {
      const float4 b = __ldg(p.bias + colf4);
      acc.x = fmaf(rs, b.x, acc.x);
      acc.y = fmaf(rs, b.y, acc.y);
      acc.z = fmaf(rs, b.z, acc.z);
      acc.w = fmaf(rs, b.w, acc.w);
    }
    if (p.accumulate) {
      const float4 o = *dst;
      acc.x += o.x;
      acc.y += o.y;
      acc.z += o.z;
      acc.w += o.w;
    }
  }
  stg_cs_f4(reinterpret_cast<float*>(dst), acc);
}

// The row pass.  SST: (col, val) and row pointers (relative to the matrix's
// first entry) in shared memory; BST: the B tile in shared memory (row pitch
// CB float4).  Entries two at a time: loads first, FMAs in storage order.
template <int CB, int EPI, bool BST, bool SST>
__device__ __forceinline__ void tile_rows(const TileParams& p, const float4* Bs, const int32_t* rp_s,
                                          const int32_t* col_s, const float* val_s, int64_t g0, int32_t n,
                                          int32_t c0, int32_t cw) {
  const int c = threadIdx.x % CB;
  if (c >= cw) return;
  constexpr int RP = kTileThreads / CB;  // rows per pass
  const float4* Bp = BST ? Bs + c : p.B + g0 * p.ldb4 + c0 + c;
  const int64_t bstride = BST ? CB : p.ldb4;
  float4* Cp = p.C + g0 * p.ldc4 + c0 + c;
  for (int32_t r = threadIdx.x / CB; r < n; r += RP) {
    int32_t e, e1;
    if (SST) {
      e = rp_s[r];
      e1 = rp_s[r + 1];
    } else {
      e = __ldg(p.row_ptr + g0 + r);
      e1 = __ldg(p.row_ptr + g0 + r + 1);
    }
    const int32_t* ci = SST ? col_s : p.col;
    const float* cv = SST ? val_s : p.vals;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float rs = 0.f;
    for (; e + 1 < e1; e += 2) {
      const int32_t k0 = SST ? ci[e] : __ldg(ci + e), k1 = SST ? ci[e + 1] : __ldg(ci + e + 1);
      const float a0 = SST ? cv[e] : __ldg(cv + e), a1 = SST ? cv[e + 1] : __ldg(cv + e + 1);
      const float4 b0 = BST ? Bp[k0 * CB] : __ldg(Bp + k0 * bstride);
      const float4 b1 = BST ? Bp[k1 * CB] : __ldg(Bp + k1 * bstride);
      fma4(acc, a0, b0);
      fma4(acc, a1, b1);
      if (EPI == 1) rs += a0, rs += a1;
    }
    if (e < e1) {
      const int32_t k0 = SST ? ci[e] : __ldg(ci + e);
      const float a0 = SST ? cv[e] : __ldg(cv + e);
      const float4 b0 = BST ? Bp[k0 * CB] : __ldg(Bp + k0 * bstride);
      fma4(acc, a0, b0);
      if (EPI == 1) rs += a0;
    }
    tile_store<EPI>(p, Cp + (int64_t)r * p.ldc4, c0 + c, acc, rs);
  }
}

template <int CB, int EPI>
__global__ void __launch_bounds__(kTileThreads) spmm_tile_kernel(const TileParams p,
                                                                 const __grid_constant__ TmaMaps maps) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  float4* Bs = reinterpret_cast<float4*>(smem);
  int32_t* rp_s = reinterpret_cast<int32_t*>(smem + p.rp_off);
  int32_t* col_s = reinterpret_cast<int32_t*>(smem + p.col_off);
  float* val_s = reinterpret_cast<float*>(smem + p.val_off);
  const int t = threadIdx.x;
  const int32_t i = (int32_t)(blockIdx.x / (uint32_t)p.tiles);
  const int32_t c0 = (int32_t)(blockIdx.x - (uint32_t)i * (uint32_t)p.tiles) * CB;
  const int32_t cw = min(CB, p.k4 - c0);
  tile_trace(p, 0);
  if (CB >= 8 && p.tma) {  // before the wait: overlaps the previous kernel's tail
    if (t == 0) {
      mbar_init(&bar, 1);
      fence_mbar_init();
    }
    if (t >= 32 && t < 32 + kTmaMaps && !(p.dbg_bits & 1)) prefetch_tensormap(&maps.m[t - 32]);
    __syncthreads();
  }
  // programmatic dependent launch: global memory only after the wait
  tile_prefetch_b(p);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  tile_trace(p, 1);

  // ---- RT1: where the matrix lives
  int64_t g0;
  int32_t n;
  if (p.row_off) {
    // read-only path: the 8-16 CTAs of an SM share the L1 line instead of
    // each warp sending its own request to the same few L2 lines
    g0 = __ldg(p.row_off + i);
    n = p.sizes ? __ldg(p.sizes + i) : (int32_t)(__ldg(p.row_off + i + 1) - g0);
  } else {  // packed layout, offsets fused into the launch
    n = __ldg(p.sizes + i);
    g0 = tile_sizes_prefix(p.sizes, i);
  }
  if (n <= 0) return;
  tile_trace(p, 2);

  // ---- B tile: n x cw float4 (row pitch CB in shared memory), by 2-D tensor
  // TMA -- popcount(n) boxes of 2^b rows, one per lane of warp 0, the higher
  // bits first (every box lands 128-byte aligned: CB >= 8) -- or by 16-byte
  // cp.async.  Columns past k are zero-filled by TMA and never stored.
  const bool bst = n <= p.cap_rows;
  const bool tma = CB >= 8 && p.tma && bst;
  BSPMM_CHECK(g0 >= 0 && n >= 0);
  // RT2 issued first (its loads are in flight while the B copies are issued;
  // they would otherwise queue behind the tile's bytes)
  int32_t z0 = 0, z1 = 0, rp0 = 0;
  if (p.rp_first) {
    z0 = __ldg(p.row_ptr + g0);
    z1 = __ldg(p.row_ptr + g0 + n);
    if (t <= n) rp0 = __ldg(p.row_ptr + g0 + t);
  }
  if (tma) {
    if (t < 32) {
      if (t == 0) mbar_arrive_expect_tx(&bar, (uint32_t)n * CB * 16u);
      __syncwarp();
      const int32_t big = n >> 8, rem = n & 255;
      for (int32_t q = t - 8; q >= 0 && q < big; q += 24)
        tma_load_2d(Bs + (size_t)q * 256 * CB, &maps.m[kTmaMaps - 1], c0 * 4, (int32_t)(g0 + q * 256), &bar);
      if (t < 8 && (rem & (1 << t))) {
        const int32_t r0 = big * 256 + (rem >> (t + 1) << (t + 1));
        tma_load_2d(Bs + (size_t)r0 * CB, &maps.m[t], c0 * 4, (int32_t)(g0 + r0), &bar);
      }
    }
  } else if (bst) {
    const float4* src = p.B + g0 * p.ldb4 + c0;
    const int32_t cells = n * cw;
    if (cw == CB) {
      for (int32_t q = t; q < cells; q += kTileThreads)
        cp_async16(Bs + q, src + (int64_t)(q / CB) * p.ldb4 + (q % CB));
    } else {
      for (int32_t q = t; q < cells; q += kTileThreads) {
        const int32_t j = q / cw, c = q - j * cw;
        cp_async16(Bs + j * CB + c, src + (int64_t)j * p.ldb4 + c);
      }
    }
    cp_async_commit();
  }
  tile_trace(p, 3);

  // ---- RT2 / RT3: row pointers, then the matrix's (col, val) run
  if (!p.rp_first) {
    z0 = __ldg(p.row_ptr + g0);
    z1 = __ldg(p.row_ptr + g0 + n);
  }
  const int32_t nz = z1 - z0;
  const bool sst = bst && nz <= p.cap_nnz;
  if (sst) {
    if (p.rp_first) {
      if (t <= n) rp_s[t] = rp0 - z0;
      for (int32_t r = t + kTileThreads; r <= n; r += kTileThreads) rp_s[r] = __ldg(p.row_ptr + g0 + r) - z0;
    } else {
      for (int32_t r = t; r <= n; r += kTileThreads) rp_s[r] = __ldg(p.row_ptr + g0 + r) - z0;
    }
    constexpr int U = 4;
    for (int32_t e = t; e < nz; e += U * kTileThreads) {
      int32_t cv[U];
      float vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int32_t ee = e + u * kTileThreads;
        cv[u] = ee < nz ? __ldg(p.col + z0 + ee) : 0;
        vv[u] = ee < nz ? __ldg(p.vals + z0 + ee) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int32_t ee = e + u * kTileThreads;
        if (ee < nz) {
          col_s[ee] = cv[u];
          val_s[ee] = vv[u];
        }
      }
    }
  }
  tile_trace(p, 4);
  if (tma) {
    __syncthreads();  // the structure in shared memory
    mbar_wait(&bar, 0);
  } else {
    if (bst) cp_async_wait_all();
    __syncthreads();
  }
  tile_trace(p, 5);

  // ---- row pass
  if (sst) tile_rows<CB, EPI, true, true>(p, Bs, rp_s, col_s, val_s, g0, n, c0, cw);
  else if (bst) tile_rows<CB, EPI, true, false>(p, Bs, rp_s, col_s, val_s, g0, n, c0, cw);
  else tile_rows<CB, EPI, false, false>(p, Bs, rp_s, col_s, val_s, g0, n, c0, cw);
  tile_trace(p, 6);
  if (p.trace && threadIdx.x == 0) {  // debug: which SM ran the tile (load-balance analysis)
    uint32_t sm;
    asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
    p.trace[(size_t)blockIdx.x * 32 + 7] = sm;
  }
}

// SparseTensor input on the tile kernel (row a-2 fused, small batches): each
// tile CTA converts its matrix's unsorted (row, col) slice to the canonical
// CSR order (row, col, original position) in shared memory -- the order of
// coo2csr.cu and of the pipeline's converter warps, so the same bits -- while
// its B tile is still landing: the raw slice is the first cp.async group, the
// tile the second, and the conversion waits only for the first.  A matrix is
// converted once per column block (L2 serves the repeats; C2: 8 CTAs x ~130
// entries).  Conversion: row histogram (shared atomics), a warp scan into the
// row pointers, scatter into the row segments (counts consumed downwards),
// then a thread per row orders its segment by the key (col << 16) | position
// (a sorting network up to 8 entries, rank counting beyond).
template <int CB>
__global__ void __launch_bounds__(kTileThreads) spmm_tile_coo_kernel(const TileParams p,
                                                                     const __grid_constant__ TmaMaps maps) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  float4* Bs = reinterpret_cast<float4*>(smem);
  int32_t* rp_s = reinterpret_cast<int32_t*>(smem + p.rp_off);
  int32_t* col_s = reinterpret_cast<int32_t*>(smem + p.col_off);
  float* val_s = reinterpret_cast<float*>(smem + p.val_off);
  int2* pr = reinterpret_cast<int2*>(smem + p.pair_off);
  float* rv = reinterpret_cast<float*>(smem + p.cval_off);
  int32_t* slot = reinterpret_cast<int32_t*>(smem + p.slot_off);
  int32_t* cnt = reinterpret_cast<int32_t*>(smem + p.cnt_off);
  const int t = threadIdx.x;
  const int32_t i = (int32_t)(blockIdx.x / (uint32_t)p.tiles);
  const int32_t c0 = (int32_t)(blockIdx.x - (uint32_t)i * (uint32_t)p.tiles) * CB;
  const int32_t cw = min(CB, p.k4 - c0);
  tile_trace(p, 0);
  const bool tma = CB >= 8 && p.tma;  // B by 2-D tensor TMA (as the CSR tile kernel), else cp.async
  if (tma) {  // before the wait: overlaps the previous kernel's tail
    if (t == 0) {
      mbar_init(&bar, 1);
      fence_mbar_init();
    }
    if (t >= 32 && t < 32 + kTmaMaps && !(p.dbg_bits & 1)) prefetch_tensormap(&maps.m[t - 32]);
    __syncthreads();
  }
  tile_prefetch_b(p);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  tile_trace(p, 1);
  // ---- RT1: where the matrix and its entries live (independent loads)
  const int64_t g0 = __ldg(p.row_off + i);
  const int32_t n = p.sizes ? __ldg(p.sizes + i) : (int32_t)(__ldg(p.row_off + i + 1) - g0);
  const int64_t z0 = __ldg(p.nnz_off + i);
  const int32_t nz = (int32_t)(__ldg(p.nnz_off + i + 1) - z0);
  if (n <= 0) return;
  if (n > p.cap_rows || nz > p.cap_nnz) {  // beyond the hints: skipped, reported by bspmm_sync
    if (t == 0) atomicOr(p.err, 64);
    return;
  }
  tile_trace(p, 2);
  // ---- the raw slice (group 0), then the B tile (group 1)
  for (int32_t e = t; e < nz; e += kTileThreads) {
    cp_async8(pr + e, p.idx + 2 * (z0 + e));
    cp_async4(rv + e, p.vals + z0 + e);
  }
  cp_async_commit();
  if (tma) {
    if (t < 32) {  // popcount(n) boxes of 2^b rows, the higher bits first
      if (t == 0) mbar_arrive_expect_tx(&bar, (uint32_t)n * CB * 16u);
      __syncwarp();
      const int32_t big = n >> 8, rem = n & 255;
      for (int32_t q = t - 8; q >= 0 && q < big; q += 24)
        tma_load_2d(Bs + (size_t)q * 256 * CB, &maps.m[kTmaMaps - 1], c0 * 4, (int32_t)(g0 + q * 256), &bar);
      if (t < 8 && (rem & (1 << t))) {
        const int32_t r0 = big * 256 + (rem >> (t + 1) << (t + 1));
        tma_load_2d(Bs + (size_t)r0 * CB, &maps.m[t], c0 * 4, (int32_t)(g0 + r0), &bar);
      }
    }
  } else {
    const float4* src = p.B + g0 * p.ldb4 + c0;
    const int32_t cells = n * cw;
    if (cw == CB) {
      for (int32_t q = t; q < cells; q += kTileThreads)
        cp_async16(Bs + q, src + (int64_t)(q / CB) * p.ldb4 + (q % CB));
    } else {
      for (int32_t q = t; q < cells; q += kTileThreads) {
        const int32_t j = q / cw, c = q - j * cw;
        cp_async16(Bs + j * CB + c, src + (int64_t)j * p.ldb4 + c);
      }
    }
  }
  cp_async_commit();  // (an empty group with TMA staging)
  for (int32_t r = t; r < n; r += kTileThreads) cnt[r] = 0;
  tile_trace(p, 3);
  cp_async_wait_group<1>();  // this thread's slice copies
  __syncthreads();
  // ---- COO -> CSR in shared memory
  for (int32_t e = t; e < nz; e += kTileThreads) atomicAdd(&cnt[pr[e].x], 1);
  __syncthreads();
  if (t < 32) {  // exclusive scan of the row counts -> rp_s (relative to the matrix's first entry)
    int32_t carry = 0;
    for (int32_t r0 = 0; r0 < n; r0 += 32) {
      const int32_t r = r0 + t;
      const int32_t v = r < n ? cnt[r] : 0;
      int32_t x = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (t >= d) x += y;
      }
      if (r < n) rp_s[r] = carry + x - v;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (t == 0) rp_s[n] = nz;
  }
  __syncthreads();
  for (int32_t e = t; e < nz; e += kTileThreads) {
    const int32_t r = pr[e].x;
    slot[rp_s[r] + atomicSub(&cnt[r], 1) - 1] = e;
  }
  __syncthreads();
  for (int32_t r = t; r < n; r += kTileThreads) {
    const int32_t s0 = rp_s[r], s1 = rp_s[r + 1], d = s1 - s0;
    if (d <= 8) {
      uint32_t key[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int32_t e = q < d ? slot[s0 + q] : 0;
        key[q] = q < d ? ((uint32_t)pr[e].y << 16) | (uint32_t)e : 0xffffffffu;
      }
#define BSPMM_TCX(a, b)                                   \
      {                                                   \
        const uint32_t lo = min(key[a], key[b]);          \
        key[b] = max(key[a], key[b]);                     \
        key[a] = lo;                                      \
      }
      if (d <= 4) {
        BSPMM_TCX(0, 1) BSPMM_TCX(2, 3) BSPMM_TCX(0, 2) BSPMM_TCX(1, 3) BSPMM_TCX(1, 2)
      } else {
        BSPMM_TCX(0, 1) BSPMM_TCX(2, 3) BSPMM_TCX(4, 5) BSPMM_TCX(6, 7)
        BSPMM_TCX(0, 2) BSPMM_TCX(1, 3) BSPMM_TCX(4, 6) BSPMM_TCX(5, 7)
        BSPMM_TCX(1, 2) BSPMM_TCX(5, 6)
        BSPMM_TCX(0, 4) BSPMM_TCX(1, 5) BSPMM_TCX(2, 6) BSPMM_TCX(3, 7)
        BSPMM_TCX(2, 4) BSPMM_TCX(3, 5)
        BSPMM_TCX(1, 2) BSPMM_TCX(3, 4) BSPMM_TCX(5, 6)
      }
#undef BSPMM_TCX
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (q < d) {
          col_s[s0 + q] = (int32_t)(key[q] >> 16);
          val_s[s0 + q] = rv[key[q] & 0xffffu];  // bitwise move
        }
      }
    } else {
      for (int32_t q = s0; q < s1; ++q) {
        const int32_t e = slot[q];
        const int32_t ce = pr[e].y;
        int32_t rank = 0;
        for (int32_t f = s0; f < s1; ++f) {
          const int32_t fe = slot[f];
          const int32_t cf = pr[fe].y;
          rank += (cf < ce) || (cf == ce && fe < e);
        }
        col_s[s0 + rank] = ce;
        val_s[s0 + rank] = rv[e];
      }
    }
  }
  tile_trace(p, 4);
  if (tma) {
    __syncthreads();  // the converted structure
    mbar_wait(&bar, 0);
  } else {
    cp_async_wait_all();  // the B tile
    __syncthreads();
  }
  tile_trace(p, 5);
  tile_rows<CB, 0, true, true>(p, Bs, rp_s, col_s, val_s, g0, n, c0, cw);
  tile_trace(p, 6);
}

// Launch geometry for a batch; false when the batch is better served by the
// persistent pipeline (more tiles than the GPU holds at once).
bool plan_tile(int32_t batch, int32_t k, int32_t max_rows, int64_t max_nnz, int32_t num_sms, int32_t cb_override,
               TileLayout* out, bool coo) {
  if (batch < 1 || k % 4 != 0) return false;
  const int32_t k4 = k / 4;
  const int64_t R = max_rows > 0 ? max_rows : kDefaultRows;
  const int64_t Z = max_nnz > 0 ? max_nnz : 8 * R;
  auto a16 = [](int64_t x) { return (x + 15) / 16 * 16; };
  auto layout = [&](int32_t cb, TileLayout& L) {
    L.cb = cb;
    L.tiles = (int32_t)ceil_div(k4, cb);
    L.units = (int64_t)batch * L.tiles;
    L.cap_rows = (int32_t)std::min<int64_t>(R, 1 << 20);
    L.cap_nnz = (int32_t)std::min<int64_t>(Z, 1 << 20);
    L.rp_off = (int32_t)a16((int64_t)L.cap_rows * cb * 16);
    L.col_off = (int32_t)(L.rp_off + a16(4LL * (L.cap_rows + 1)));
    L.val_off = (int32_t)(L.col_off + a16(4LL * L.cap_nnz));
    L.smem = (int32_t)(L.val_off + a16(4LL * L.cap_nnz));
    if (coo) {  // SparseTensor conversion scratch: raw pairs, raw values, slots, row counters
      L.pair_off = L.smem;
      L.cval_off = (int32_t)(L.pair_off + a16(8LL * L.cap_nnz));
      L.slot_off = (int32_t)(L.cval_off + a16(4LL * L.cap_nnz));
      L.cnt_off = (int32_t)(L.slot_off + a16(4LL * L.cap_nnz));
      L.smem = (int32_t)(L.cnt_off + a16(4LL * (L.cap_rows + 1)));
    }
    // resident CTAs per SM: 16 by threads (2048 / 128), fewer by shared memory
    // (228 KB per SM, 1 KB reserved per CTA)
    L.per_sm = (int32_t)std::min<int64_t>(16, 233472 / (L.smem + 1024 + 64));
  };
  TileLayout L{};
  if (cb_override > 0) {
    int32_t cb = 1;
    while (cb < cb_override && cb < 32) cb <<= 1;
    layout(cb, L);
  } else {
    // widest tiles that still give >= 8 tiles per SM (overlap between the CTAs
    // of an SM), and a B tile of at most 32 KB, but no narrower than 2 float4
    // (32-byte rows) -- with cp.async staging the narrow blocks beat the
    // pipeline on small batches (config 2: cb 2 = 800 tiles 3.38 us, cb 4 3.58,
    // cb 1 3.90, the pipeline 3.81; config 4: cb 8 6.66, cb 16 6.98, cb 4 8.51;
    // tools/probe/tile_balance.py)
    int32_t cb = 1;
    while (cb < 32 && cb < k4) cb <<= 1;
    layout(cb, L);
    while (cb > 2 && (L.units < 8LL * num_sms || R * cb * 16 > 32768)) {
      cb >>= 1;
      layout(cb, L);
    }
    if (cb < 2) return false;
  }
  if (L.smem > 200 * 1024 || L.per_sm < 1) return false;
  // the conversion's 16-bit sort keys: positions and columns below 2^16
  if (coo && (L.cap_nnz >= 65536 || L.cap_rows >= 65536)) return false;
  // one wave: every tile resident at once (beyond that the persistent
  // pipeline streams better, e.g. config 5)
  if (cb_override <= 0 && L.units > (int64_t)L.per_sm * num_sms) return false;
  *out = L;
  return true;
}

template <int CB, int EPI>
static cudaError_t launch_tile_t(const TileParams& tp, const TmaMaps& maps, const TileLayout& L, cudaStream_t s) {
  auto kern = spmm_tile_kernel<CB, EPI>;
  static thread_local int configured[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (L.smem > 47 * 1024 && configured[dev & 63] < L.smem) {  // dynamic + static above the 48 KB default
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.smem);
    if (e != cudaSuccess) return e;
    configured[dev & 63] = L.smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)L.units);
  cfg.blockDim = dim3(kTileThreads);
  cfg.dynamicSmemBytes = L.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, tp, maps);
}

template <int EPI>
static cudaError_t launch_tile_e(const TileParams& tp, const TmaMaps& m, const TileLayout& L, cudaStream_t s) {
  switch (L.cb) {
    case 1: return launch_tile_t<1, EPI>(tp, m, L, s);
    case 2: return launch_tile_t<2, EPI>(tp, m, L, s);
    case 4: return launch_tile_t<4, EPI>(tp, m, L, s);
    case 8: return launch_tile_t<8, EPI>(tp, m, L, s);
    case 16: return launch_tile_t<16, EPI>(tp, m, L, s);
    default: return launch_tile_t<32, EPI>(tp, m, L, s);
  }
}

template <int CB>
static cudaError_t launch_tile_coo_t(const TileParams& tp, const TmaMaps& m, const TileLayout& L, cudaStream_t s) {
  auto kern = spmm_tile_coo_kernel<CB>;
  static thread_local int configured[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (L.smem > 47 * 1024 && configured[dev & 63] < L.smem) {  // dynamic + static above the 48 KB default
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.smem);
    if (e != cudaSuccess) return e;
    configured[dev & 63] = L.smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)L.units);
  cfg.blockDim = dim3(kTileThreads);
  cfg.dynamicSmemBytes = L.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, tp, m);
}

cudaError_t launch_spmm_tile(const CsrArgs& a, const TileLayout& L, cudaStream_t s) {
  if (L.units == 0) return cudaSuccess;
  if (L.units > 0x7fffffffLL) return cudaErrorInvalidValue;
  TileParams tp;
  tp.batch = a.batch;
  tp.k4 = a.k / 4;
  tp.tiles = L.tiles;
  tp.cap_rows = L.cap_rows;
  tp.cap_nnz = L.cap_nnz;
  tp.rp_off = L.rp_off;
  tp.col_off = L.col_off;
  tp.val_off = L.val_off;
  tp.row_off = a.row_off;
  tp.sizes = a.sizes;
  tp.row_ptr = a.row_ptr;
  tp.col = a.col;
  tp.vals = a.vals;
  tp.B = reinterpret_cast<const float4*>(a.B);
  tp.ldb4 = a.ldb / 4;
  tp.C = reinterpret_cast<float4*>(a.C);
  tp.ldc4 = a.ldc / 4;
  tp.bias = reinterpret_cast<const float4*>(a.bias);
  tp.accumulate = a.accumulate;
  tp.trace = a.trace;
  // B by 2-D tensor TMA where that applies (the handle's descriptors for box
  // width 4 * cb, a 128-byte shared row pitch; column blocks of >= 8 float4),
  // else by 16-byte cp.async (debug bit 32768: always cp.async).  With the
  // pre-wait prefetch the tile is an L2 hit and TMA's few bulk copies leave
  // the LSU to the structure round trips: C4 5.62-5.65 vs 5.83-5.85 us (the
  // order was the reverse before the prefetch: 6.87 vs 6.70 us)
  tp.tma = (a.maps != nullptr && L.cb >= 8 && !(a.dbg & 32768)) ? 1 : 0;
  tp.rp_first = (a.dbg & 65536) ? 0 : 1;
  tp.dbg_bits = ((a.dbg & 16) ? 1 : 0) | ((a.dbg & (1 << 26)) ? 2 : 0);
  tp.nnz_off = a.coo_nnz_off;
  tp.idx = a.coo_idx;
  tp.pair_off = L.pair_off;
  tp.cval_off = L.cval_off;
  tp.slot_off = L.slot_off;
  tp.cnt_off = L.cnt_off;
  tp.err = a.err;
  tp.b_lo = a.b_lo;
  tp.b_hi = a.b_hi;
  for (int q = 0; q < 3; ++q) {
    tp.s_lo[q] = a.s_lo[q];
    tp.s_hi[q] = a.s_hi[q];
  }
  static const TmaMaps no_maps{};
  const TmaMaps& m = a.maps ? *a.maps : no_maps;
  if (a.coo_nnz_off) {  // SparseTensor input: the converting variant (row_off required)
    if (!a.row_off || !a.err || a.bias != nullptr || a.accumulate != 0) return cudaErrorInvalidValue;
    switch (L.cb) {
      case 1: return launch_tile_coo_t<1>(tp, m, L, s);
      case 2: return launch_tile_coo_t<2>(tp, m, L, s);
      case 4: return launch_tile_coo_t<4>(tp, m, L, s);
      case 8: return launch_tile_coo_t<8>(tp, m, L, s);
      case 16: return launch_tile_coo_t<16>(tp, m, L, s);
      default: return launch_tile_coo_t<32>(tp, m, L, s);
    }
  }
  if (a.bias != nullptr || a.accumulate != 0) return cudaErrorInvalidValue;  // no GCN epilogue here (gcn_fused.cu)
  return launch_tile_e<0>(tp, m, L, s);
}

}  // namespace bspmm
