// spmm_csr.cu — the batched CSR SpMM kernel for sm_100a (hot-path rows a-4,
// a-5, a-6).
//
// What it computes (PAPER.md Fig. algo:code_swa_spmm_csr, lines 196-207,
// batched as in §IV-C): for every matrix i, row r < n_i and
// column c < k
//     C[g][c] = sum_{e in row g} vals[e] * B[row_off[i] + col[e]][c],
// g = row_off[i] + r, accumulated as fp32 FMA in CSR storage order from +0.
//
// How (B200-first; the paper's P100 design is prior art):
//  * persistent CTAs walk units u = (matrix i, k-tile t) with stride grid;
//  * warp 0 is the PRODUCER: it prefetches unit metadata 32 units at a time
//    (one lane per unit), then per unit waits for a free ring stage and
//    stages B_i[:, tile] into shared memory with TMA bulk copies
//    (cp.async.bulk, one copy when the tile is the whole contiguous B_i,
//    else one per row) and the unit's CSR structure (row pointers, (col, val)
//    pairs) with cp.async, all completing on the stage's "full" mbarrier;
//  * warps 1..W are CONSUMERS: a sub-warp of `lanes` lanes owns one row at a
//    time (SWA; row ownership means no atomics, :170), each
//    lane owns float4 column chunks (the paper's lane-strided columns
//    j = lane, lane + subWarp, ..., :204, widened to 128-bit), reads B from
//    shared memory, accumulates in registers and writes the C row with
//    128-bit streaming stores.  Empty rows store +0 (no init launch,
//    PAPER.md:220-222).  Then the warp arrives on the stage's "empty" barrier;
//  * a unit whose tile or structure exceeds the stage capacity is computed
//    straight from global memory (the paper's no-shared-memory case 3,
//    PAPER.md:249-252), decided per unit on the device.
#include <cstdint>

#include "internal.h"
#include "ptx.cuh"

namespace bspmm {

struct SpmmParams {
  int64_t units;
  int32_t tiles, kt, k;
  int32_t stages, stage_b, stage_s, lanes;
  const int64_t* __restrict__ row_off;
  const int32_t* __restrict__ sizes;
  const int32_t* __restrict__ row_ptr;
  const int32_t* __restrict__ col;
  const float* __restrict__ vals;
  const float* __restrict__ B;
  int64_t ldb;
  float* __restrict__ C;
  int64_t ldc;
  unsigned long long* trace;  // debug: per-CTA phase timestamps (globaltimer ns), or null
  int32_t dbg;                // debug bits: 1 skip C stores, 2 unit direct, 8 consumer work x4 (experiments)
  int32_t tma2d;              // 1: full k-tiles staged with 2-D tensor TMA (maps valid)
  int32_t sbulk;              // 1: col / vals / row_ptr bases are 16-byte aligned (bulk-copy the CSR slice)
  int32_t slice_lsu;          // 1: CSR slice by 16-byte cp.async instead of TMA bulk (small problems)
  const float* __restrict__ bias;  // GCN epilogue (NEXT-1): C += rowsum(A) (x) bias[c0..], or null
  int32_t accumulate;              // GCN epilogue: C += previous C (channel accumulation)
  unsigned long long* sched;       // dynamic schedule ticket counter (self-resetting), or null (static)
  // fused COO mode (bspmm_coo): the unit's SparseTensor slice is converted to
  // CSR in shared memory by the consumers (row a-2 inside the SpMM launch)
  const int64_t* __restrict__ nnz_off;
  const int32_t* __restrict__ idx;   // [nnz][2] (row, col) local pairs
  int* err;                          // device flag: bit 64 = a unit exceeded the stage (hint too small)
  int32_t cvt_warps;                 // fused COO mode: converter warps (the last ones of the CTA)
  int32_t coo_rows;                  // fused COO mode: row capacity of a stage (the hinted max_rows)
  int32_t mc;                        // NEXT-4b: C is a multicast address (EPI == 2: multimem.st stores)
  // SDDMM mode (EPI == 3, NEXT-2 backward): sd_out[e] = <G[row_e], B[col_e]>
  // over the staged B_i, whole-row units (tiles == 1); C is not written
  const float* __restrict__ G;
  int64_t ldg;
  float* __restrict__ sd_out;
  // pre-wait L2 prefetch (few units per CTA): B's and the structure arrays'
  // allocations (CSR row_ptr, col, vals; COO -, idx, vals); b_hi == 0: off
  uint64_t b_lo, b_hi;
  uint64_t s_lo[3], s_hi[3];
  uint64_t g_lo, g_hi;  // SDDMM mode: grad_C's allocation (its rows are prefetched too)
};

// GCN epilogue (NEXT-1, PAPER.md Fig. algo:graph_conv_batched): A (U + 1 b^T)
// = A U + rowsum(A) b^T, so the bias add folds into the SpMM as rs * b after
// the storage-order sum; channels accumulate into C.
template <int EPI, bool VEC>
__device__ __forceinline__ void epilogue(const SpmmParams& p, float4& acc, float rs, int64_t colf, const float* cptr) {
  if (EPI != 1) return;
  if (p.bias) {
    if (VEC) {
      const float4 b = ldg_nc_f4(p.bias + colf);
      acc.x = fmaf(rs, b.x, acc.x);
      acc.y = fmaf(rs, b.y, acc.y);
      acc.z = fmaf(rs, b.z, acc.z);
      acc.w = fmaf(rs, b.w, acc.w);
    } else {
      acc.x = fmaf(rs, __ldg(p.bias + colf), acc.x);
    }
  }
  if (p.accumulate) {
    if (VEC) {
      const float4 o = *reinterpret_cast<const float4*>(cptr);
      acc.x += o.x;
      acc.y += o.y;
      acc.z += o.z;
      acc.w += o.w;
    } else {
      acc.x += *cptr;
    }
  }
}

// a-6 store of one chunk: streaming st.global, or (EPI == 2, NEXT-4b) one
// multimem store that writes the row of C into every GPU of the
// multicast team -- the all-gather of the sharded C done by the store itself.
template <int EPI, bool VEC>
__device__ __forceinline__ void store_c(const SpmmParams& p, float* ptr, const float4& acc) {
  if (EPI == 2) {
    if (VEC) mm_st_f4(ptr, acc);
    else mm_st_f1(ptr, acc.x);
  } else {
    if (VEC) stg_cs_f4(ptr, acc);
    else stg_cs_f1(ptr, acc.x);
  }
}

// Stage layout of a unit's CSR slice, after the B tile: three int32 arrays
// (col, vals, row pointers), each in a region of 16 + 4*count bytes rounded
// to 16, with element 0 at byte (first & 3) * 4 so that the 16-byte-aligned
// interior of the source lands 16-byte aligned (TMA bulk copy).
__device__ __forceinline__ int64_t i64min(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int32_t slice_region(int64_t count) { return (int32_t)((16 + 4 * count + 15) & ~15LL); }
__host__ __device__ __forceinline__ int64_t slice_bytes(int64_t nnz, int64_t n) {
  return 2LL * slice_region(nnz) + slice_region(n + 1);
}
// fused COO mode, after the CSR slice: raw (row, col) pairs (element 0 at pair
// (first & 1)), raw values (element 0 at (first & 3)), per-row cursors, slots
__host__ __device__ __forceinline__ int64_t al16(int64_t x) { return (x + 15) & ~15LL; }
__host__ __device__ __forceinline__ int64_t coo_raw_off(int64_t nnz, int64_t n) { return al16(slice_bytes(nnz, n)); }
__host__ __device__ __forceinline__ int64_t coo_pairs_bytes(int64_t nnz) { return al16(8 * (nnz + 1)); }
__host__ __device__ __forceinline__ int64_t coo_vals_bytes(int64_t nnz) { return al16(4 * (nnz + 3)); }
// ... + slots [nnz]; the per-row counters live at a FIXED place, the end of
// the stage's structure region (capacity `cap` rows): they are zeroed once at
// kernel start and left at zero by every conversion (counted up by the row
// histogram, back down by the scatter)
__host__ __device__ __forceinline__ int64_t coo_cursor_bytes(int64_t cap) { return al16(4 * (cap + 1)); }
__host__ __device__ __forceinline__ int64_t coo_stage_bytes(int64_t nnz, int64_t n, int64_t cap) {
  return coo_raw_off(nnz, n) + coo_pairs_bytes(nnz) + coo_vals_bytes(nnz) + al16(4 * nnz) + coo_cursor_bytes(cap);
}

// trace slots per CTA (bspmm_set_trace): 0 entry, 1 after PDL wait, 2 producer has unit-0 row
// offsets, 3 producer has unit-0 structure offsets, 4 producer issued its last unit, 5 first
// consumer warp saw unit 0 land, 6 first consumer warp finished its last unit, 7 CTA exit,
// 8 first consumer warp finished unit 0
constexpr int kTraceSlots = 32;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define BSPMM_TRACE(p, slot) \
  do {                      \
    if (p.trace) p.trace[(size_t)blockIdx.x * kTraceSlots + (slot)] = gtime(); \
  } while (0)

// CTA size cap per chunk count: 16 consumer warps fit the register budget with
// up to 2 chunks per lane; 4 chunks need ~128 registers -> 15 consumer warps
constexpr int kMaxThreads(int ch) { return ch >= 4 ? 512 : 544; }
constexpr int kMaxRegs(int ch) { return ch >= 4 ? 128 : 120; }
// fused COO mode: kCooWarps warps (5 per SM sub-partition: 96 registers)
constexpr int kMaxThreadsK(int ch, bool coo) { return coo ? 32 * kCooWarps : kMaxThreads(ch); }
constexpr int kMaxRegsK(int ch, bool coo) { return coo ? 96 : kMaxRegs(ch); }

struct __align__(16) UnitHdr {
  int64_t g0;     // first global row of the matrix
  int32_t n;      // rows (n_i)
  int32_t nz0;    // absolute position of the matrix's first entry
  int32_t nnz;    // entries of the matrix
  int32_t c0;     // first column of the tile
  int32_t kw;     // tile width (ragged last tile)
  int32_t flags;  // bit0: B tile staged in smem; bit1: CSR structure staged in smem
};
static_assert(sizeof(UnitHdr) == kHdrBytes, "header size");

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

// unit metadata, one unit per producer lane
struct Meta {
  int64_t g0;
  int32_t n, c0, kw, nz0, nz1;
};

// Fused batch-offset builder (row a-1 inside the SpMM, row_off == null):
// the prefix P(i) = sum_{m<i} sizes[m] for this lane's unit base + lane*G,
// from a warp scan of per-lane segment sums; `carry` holds P at the batch
// start and advances to P at the next batch's start.
__device__ __forceinline__ int64_t fused_prefix(const SpmmParams& p, int64_t base, int64_t G, int lane,
                                                int64_t& carry) {
  const int64_t bmax = p.units / p.tiles;  // matrices
  auto mat = [&](int64_t u) { return u < p.units ? u / p.tiles : bmax; };
  const int64_t i0 = mat(base + (int64_t)lane * G);
  int64_t i1 = mat(base + (int64_t)(lane + 1) * G);
  // a lane's segment feeds only the lanes after it (exclusive scan) and the
  // next batch's carry: in the CTA's last batch, segments from the last valid
  // unit on are not needed (C4: one unit per CTA -> no loads at all)
  if (base + 32 * G >= p.units && (base + (int64_t)(lane + 1) * G) >= p.units) i1 = i0;
  // segment sum with many loads in flight: 16-byte loads, 8 per step, split partial sums
  int64_t seg = 0;
  int64_t m = i0;
  const bool al = (reinterpret_cast<uintptr_t>(p.sizes) & 15u) == 0;
  if (al) {
    for (; m < i1 && (m & 3); ++m) seg += __ldg(p.sizes + m);
    const int4* v4 = reinterpret_cast<const int4*>(p.sizes + m);
    const int64_t nv = (i1 - m) >> 2;
    int64_t q = 0;
    int32_t s0 = 0, s1 = 0;
    for (; q + 8 <= nv; q += 8) {
      int4 t[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) t[r] = __ldg(v4 + q + r);
#pragma unroll
      for (int r = 0; r < 8; r += 2) {
        s0 += t[r].x + t[r].y + t[r].z + t[r].w;
        s1 += t[r + 1].x + t[r + 1].y + t[r + 1].z + t[r + 1].w;
      }
      seg += (int64_t)s0 + s1;  // int32 partials per 32 sizes, widened (sizes < 2^31 each)
      s0 = s1 = 0;
    }
    for (; q < nv; ++q) {
      const int4 t = __ldg(v4 + q);
      seg += (int64_t)t.x + t.y + t.z + t.w;
    }
    m += nv << 2;
  }
  for (; m < i1; ++m) seg += __ldg(p.sizes + m);
  int64_t x = seg;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  const int64_t pre = carry + x - seg;
  carry += __shfl_sync(0xffffffffu, x, 31);
  return pre;
}
// sum of sizes[0 .. i0) over the warp (i0 < grid: a handful per lane): the
// first 8 loads per lane are all in flight before any add (one round trip)
__device__ __forceinline__ int64_t warp_sizes_sum(const int32_t* __restrict__ sizes, int64_t i0, int lane) {
  int32_t v[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int64_t m = lane + 32 * q;
    v[q] = m < i0 ? __ldg(sizes + m) : 0;
  }
  int64_t s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += v[q];
  for (int64_t m = lane + 256; m < i0; m += 32) s += __ldg(sizes + m);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
  return s;
}
__device__ __forceinline__ int64_t fused_prefix_start(const SpmmParams& p, int lane) {
  return warp_sizes_sum(p.sizes, (int64_t)blockIdx.x / p.tiles, lane);  // matrices before this CTA's first unit
}

// round trip 1 for unit uu: row offset (or the fused prefix g0f), rows, tile
template <bool COO>
__device__ __forceinline__ void meta_rt1(const SpmmParams& p, int64_t uu, Meta& m, int64_t g0f = -1) {
  if (uu < p.units) {
    const int64_t i = uu / p.tiles;
    const int32_t t = (int32_t)(uu - i * p.tiles);
    m.g0 = p.row_off ? p.row_off[i] : g0f;
    m.n = p.sizes ? p.sizes[i] : (int32_t)(p.row_off[i + 1] - m.g0);
    m.c0 = t * p.kt;
    m.kw = min(p.kt, p.k - m.c0);
    if (COO) {  // fused COO mode: the entry range comes with round trip 1
      m.nz0 = (int32_t)p.nnz_off[i];
      m.nz1 = (int32_t)p.nnz_off[i + 1];
    }
  } else {
    m.g0 = 0; m.n = 0; m.c0 = 0; m.kw = 0;
  }
}
// round trip 2: the matrix's entry range (depends on round trip 1)
template <bool COO>
__device__ __forceinline__ void meta_rt2(const SpmmParams& p, int64_t uu, Meta& m) {
  if (COO) return;  // fused COO mode: no row pointers
  if (uu < p.units) {
    m.nz0 = p.row_ptr[m.g0];
    m.nz1 = p.row_ptr[m.g0 + m.n];
  } else {
    m.nz0 = 0; m.nz1 = 0;
  }
}

// Early B tile of a CTA's FIRST unit (latency-bound launches): consumer warp
// 0 -- idle until the first unit lands -- loads the unit's row range itself
// and issues its B tile at once, on a barrier of its own (bfull), while the
// producer is still on the structure round trip (row_ptr) and the CSR slice.
// The B tile is the long pole of a unit's landing (C4: 100 KB per CTA).
// Conditions are evaluated identically by the producer (which then skips the
// tile) and by consumer warp 0.
__device__ __forceinline__ uint64_t* early_bar(const SpmmParams& p, unsigned char* smem) {
  return reinterpret_cast<uint64_t*>(smem + p.stages * (kHdrBytes + 16));
}
// fused COO mode: per-stage barrier of the raw slice (+ header)
__device__ __forceinline__ uint64_t* sfull_bar(const SpmmParams& p, unsigned char* smem) {
  return reinterpret_cast<uint64_t*>(smem + p.stages * (kHdrBytes + 16) + 8);
}
// fused COO mode: per-stage "converted" barrier (one arrival per converter warp)
__device__ __forceinline__ uint64_t* cvt_bar(const SpmmParams& p, unsigned char* smem) {
  return reinterpret_cast<uint64_t*>(smem + p.stages * (kHdrBytes + 24) + 8);
}
template <bool VEC, bool COO>
__device__ __forceinline__ bool early_b_ok(const SpmmParams& p, int32_t n, int32_t kw) {
  // whole contiguous B_i only (one 1-D bulk copy): with k-tiles (2-D boxes) it
  // measured slower (C3 12.45 vs 12.16 us), whole rows faster (C4 7.9 -> 7.05 us)
  // (not in fused COO mode: its consumer kernel spills with the extra path, C3 19.8 -> 25 us)
  return VEC && !COO && !p.sched && !(p.dbg & (2 | 4)) && n > 0 &&
         (int64_t)n * kw * 4 <= p.stage_b && kw == p.ldb;
}

// consumer warp 0's side of the early B tile, out of line so that it does not
// add to the consumer loop's register allocation (arguments by value: no
// local copy of the parameter block).  Must agree with early_b_ok.
__device__ __noinline__ void early_b_issue(const int64_t* __restrict__ row_off, const int32_t* __restrict__ sizes,
                                           const float* __restrict__ B, int64_t ldb, int32_t tiles, int32_t kt,
                                           int32_t k, int32_t stage_b, unsigned long long* trace, uint64_t* eb,
                                           unsigned char* st) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x / tiles;
  const int32_t t = (int32_t)((int64_t)blockIdx.x - i * tiles);
  // packed layout with offsets fused: g0 = sum of the sizes before matrix i
  const int32_t ni = sizes ? __ldg(sizes + i) : 0;
  const int64_t g0 = row_off ? row_off[i] : warp_sizes_sum(sizes, i, lane);
  const int32_t n = sizes ? ni : (int32_t)(row_off[i + 1] - g0);
  const int32_t c0 = t * kt, kw = min(kt, k - c0);
  if (!(n > 0 && (int64_t)n * kw * 4 <= stage_b && kw == ldb)) return;
  if (lane == 0) {
    mbar_arrive_expect_tx(eb, (uint32_t)n * (uint32_t)kw * 4u);
    bulk_g2s_hint(st, B + g0 * ldb + c0, (uint32_t)n * (uint32_t)kw * 4u, eb, policy_evict_first());
    if (trace) trace[(size_t)blockIdx.x * kTraceSlots + 15] = gtime();
  }
}

// Stage unit j of this CTA (metadata already known): wait for its ring stage,
// TMA/cp.async the B tile and CSR slice, publish the header, arrive on "full".
template <bool VEC, bool COO>
__device__ __forceinline__ void issue_unit(const SpmmParams& p, const TmaMaps& maps, unsigned char* smem, int j,
                                           int64_t g0, int32_t n, int32_t c0, int32_t kw, int32_t nz0, int32_t nnz,
                                           bool b_early = false) {
  UnitHdr* hdr = reinterpret_cast<UnitHdr*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * kHdrBytes);
  uint64_t* empty = full + p.stages;
  unsigned char* ring = smem + ring_prefix_bytes(p.stages);
  const int32_t stage_bytes = p.stage_b + p.stage_s;
  const int lane = threadIdx.x & 31;
  const uint64_t pol = policy_evict_first();
    const int s = j % p.stages;
    const uint32_t phase = (uint32_t)(j / p.stages) & 1u;
    mbar_wait(&empty[s], phase ^ 1u);
    if (j == 0 && lane == 0) BSPMM_TRACE(p, 9);
    if (j < 3 && lane == 0) BSPMM_TRACE(p, 16 + 4 * j);
    unsigned char* st = ring + (size_t)s * stage_bytes;
    const float* bsrc = p.B + g0 * p.ldb + c0;
    unsigned char* sreg = st + p.stage_b;
    if (COO) {  // fused COO mode: B tile (on full[s]) + the raw SparseTensor slice (on sfull[s])
      uint64_t* sfull = sfull_bar(p, smem);
      const bool fits = (int64_t)n * kw * 4 <= p.stage_b && n <= p.coo_rows &&
                        coo_stage_bytes(nnz, n, p.coo_rows) <= p.stage_s;
      if (fits && n > 0) {
        if (lane == 0) mbar_expect_tx(&full[s], (uint32_t)n * (uint32_t)kw * 4u);
        __syncwarp();
        if (kw == p.ldb) {
          if (lane == 3) bulk_g2s_hint(st, bsrc, (uint32_t)n * (uint32_t)kw * 4u, &full[s], pol);
        } else if (p.tma2d && kw == p.kt) {
          const int32_t big = n >> 8, rem = n & 255;
          for (int32_t q = lane - 4; q >= 0 && q < big && lane < 16; q += 12)
            tma_load_2d(st + (size_t)q * 256 * kw * 4, &maps.m[kTmaMaps - 1], c0, (int32_t)(g0 + q * 256), &full[s]);
          const int b = lane - 16;
          if (b >= 0 && b < 8 && (rem & (1 << b))) {
            const int32_t r0 = big * 256 + (rem >> (b + 1) << (b + 1));
            tma_load_2d(st + (size_t)r0 * kw * 4, &maps.m[b], c0, (int32_t)(g0 + r0), &full[s]);
          }
        } else {
          for (int r = lane; r < n; r += 32)
            bulk_g2s_hint(st + (size_t)r * kw * 4, bsrc + (int64_t)r * p.ldb, (uint32_t)kw * 4u, &full[s], pol);
        }
        unsigned char* raw = sreg + coo_raw_off(nnz, n);
        int32_t* dpair = reinterpret_cast<int32_t*>(raw) + 2 * (nz0 & 1);
        int32_t* dval = reinterpret_cast<int32_t*>(raw + coo_pairs_bytes(nnz)) + (nz0 & 3);
        const int32_t* spair = p.idx + 2 * (int64_t)nz0;
        const int32_t* sval = reinterpret_cast<const int32_t*>(p.vals) + nz0;
        if (p.sbulk) {  // 16-byte interiors, 8-/4-byte edges
          const int32_t pa = min(nnz, nz0 & 1), pb = pa + ((nnz - pa) & ~1);  // pairs [pa, pb): 16-byte chunks
          for (int32_t q = lane; q < ((pb - pa) >> 1); q += 32) cp_async16(dpair + 2 * (pa + 2 * q), spair + 2 * (pa + 2 * q));
          if (lane == 0 && pa == 1 && nnz > 0) cp_async8(dpair, spair);
          if (lane == 1 && pb < nnz) cp_async8(dpair + 2 * pb, spair + 2 * pb);
          const int32_t va = (int32_t)(i64min(nnz, (4 - (nz0 & 3)) & 3)), vb = va + ((nnz - va) & ~3);
          for (int32_t q = lane; q < ((vb - va) >> 2); q += 32) cp_async16(dval + va + 4 * q, sval + va + 4 * q);
          if (lane >= 24 && lane < 24 + va) cp_async4(dval + (lane - 24), sval + (lane - 24));
          if (lane >= 28 && vb + (lane - 28) < nnz) cp_async4(dval + vb + (lane - 28), sval + vb + (lane - 28));
        } else {
          for (int32_t e = lane; e < nnz; e += 32) {
            cp_async4(dpair + 2 * e, spair + 2 * e);
            cp_async4(dpair + 2 * e + 1, spair + 2 * e + 1);
            cp_async4(dval + e, sval + e);
          }
        }
      } else if (!fits && lane == 0) {
        atomicOr(p.err, 64);  // planner hint too small: the unit is skipped, reported by bspmm_sync
      }
      if (lane == 0) {
        UnitHdr h;
        h.g0 = g0; h.n = n; h.nz0 = nz0; h.nnz = nnz; h.c0 = c0; h.kw = kw;
        h.flags = fits ? 3 : 4;
        hdr[s] = h;
        mbar_arrive(&sfull[s]);
        mbar_arrive(&full[s]);
      }
      cp_async_arrive_noinc(&sfull[s]);
      return;
    }
    // a unit is staged whole (tile + structure) or not at all (read from global memory)
    const bool bst = (int64_t)n * kw * 4 <= p.stage_b && slice_bytes(nnz, n) <= p.stage_s && !(p.dbg & 2);
    const bool sst = bst;
    if (bst) {
      // a-4 + the CSR slice. Lane 0 announces every TMA byte of the unit once,
      // then issues the copies; the <= 3 unaligned head/tail elements of each
      // slice array go by 4-byte cp.async on lanes 0..17.
      const int32_t a_col = p.sbulk ? (int32_t)(i64min(nz0 + nnz, (nz0 + 3) & ~3LL) - nz0) : nnz;
      const int32_t b_col = p.sbulk ? max(a_col, (int32_t)(((nz0 + nnz) & ~3LL) - nz0)) : nnz;
      const int64_t r_lo = g0, r_cnt = n + 1;
      const int32_t a_rp = p.sbulk ? (int32_t)(i64min(r_lo + r_cnt, (r_lo + 3) & ~3LL) - r_lo) : (int32_t)r_cnt;
      const int32_t b_rp = p.sbulk ? max(a_rp, (int32_t)(((r_lo + r_cnt) & ~3LL) - r_lo)) : (int32_t)r_cnt;
      int32_t* dcol = reinterpret_cast<int32_t*>(sreg) + (nz0 & 3);
      int32_t* dval = reinterpret_cast<int32_t*>(sreg + slice_region(nnz)) + (nz0 & 3);
      int32_t* drp = reinterpret_cast<int32_t*>(sreg + 2 * slice_region(nnz)) + (r_lo & 3);
      const bool b_bulk = VEC && n > 0 && !b_early;  // (an early tile is already in flight)
      // lane 0 announces every TMA byte of the unit, then each copy is issued
      // by its own lane: on a cold start every issue stalls its thread ~0.1 us
      // (measured with tools/trace.py), so serial issue from one lane cost
      // ~1 us per unit; spread over lanes the stalls overlap
      // the CSR slice's 16-byte-aligned interior: TMA bulk copies for streaming
      // batches (fewest instructions), 16-byte cp.async (LSU path) for small
      // latency-bound batches, where the SM's TMA front-end accepting copies one
      // at a time on a cold start is on the critical path (tools/trace.py)
      const bool slice_tma = p.sbulk && !p.slice_lsu;
      if (lane == 0) {
        uint32_t tx = b_bulk ? (uint32_t)n * (uint32_t)kw * 4u : 0u;
        if (slice_tma) tx += 2u * 4u * (uint32_t)(b_col - a_col) + 4u * (uint32_t)(b_rp - a_rp);
        if (tx) mbar_expect_tx(&full[s], tx);
      }
      __syncwarp();
      auto issue_b = [&]() {
      if (b_bulk) {  // TMA: whole contiguous B_i (1-D), a full k-tile (2-D boxes), else one bulk copy per row
        if (kw == p.ldb) {
          if (lane == 3) bulk_g2s_hint(st, bsrc, (uint32_t)n * (uint32_t)kw * 4u, &full[s], pol);
        } else if (p.tma2d && kw == p.kt) {
          // boxes: floor(n / 256) of 256 rows (lanes 4..), then the set bits of n % 256 (lanes 16 + b)
          const int32_t big = n >> 8, rem = n & 255;
          for (int32_t q = lane - 4; q >= 0 && q < big && lane < 16; q += 12)
            tma_load_2d(st + (size_t)q * 256 * kw * 4, &maps.m[kTmaMaps - 1], c0, (int32_t)(g0 + q * 256), &full[s]);
          const int b = lane - 16;
          if (b >= 0 && b < 8 && (rem & (1 << b))) {
            const int32_t r0 = big * 256 + (rem >> (b + 1) << (b + 1));
            tma_load_2d(st + (size_t)r0 * kw * 4, &maps.m[b], c0, (int32_t)(g0 + r0), &full[s]);
          }
        } else {
          for (int r = lane; r < n; r += 32)
            bulk_g2s_hint(st + (size_t)r * kw * 4, bsrc + (int64_t)r * p.ldb, (uint32_t)kw * 4u, &full[s], pol);
        }
      }
      };
      // the B tile first: it is the long pole of a unit's landing (C4: 100 KB;
      // 7.9 vs 8.2 us, C5 810 vs 817 us)
      issue_b();
      if (p.trace) __syncwarp();
      if (j < 3 && lane == 0) BSPMM_TRACE(p, 18 + 4 * j);
      if (slice_tma) {
        if (b_col > a_col) {
          if (lane == 0) bulk_g2s(dcol + a_col, p.col + nz0 + a_col, 4u * (uint32_t)(b_col - a_col), &full[s]);
          if (lane == 1) bulk_g2s(dval + a_col, p.vals + nz0 + a_col, 4u * (uint32_t)(b_col - a_col), &full[s]);
        }
        if (lane == 2 && b_rp > a_rp)
          bulk_g2s(drp + a_rp, p.row_ptr + r_lo + a_rp, 4u * (uint32_t)(b_rp - a_rp), &full[s]);
      } else if (p.sbulk) {
        const int32_t ncol4 = (b_col - a_col) >> 2, nrp4 = (b_rp - a_rp) >> 2;
        for (int32_t q = lane; q < ncol4; q += 32) {
          cp_async16(dcol + a_col + 4 * q, p.col + nz0 + a_col + 4 * q);
          cp_async16(dval + a_col + 4 * q, p.vals + nz0 + a_col + 4 * q);
        }
        for (int32_t q = lane; q < nrp4; q += 32) cp_async16(drp + a_rp + 4 * q, p.row_ptr + r_lo + a_rp + 4 * q);
      }
      if (p.trace) __syncwarp();
      if (j < 3 && lane == 0) BSPMM_TRACE(p, 17 + 4 * j);
      if (j == 0 && lane == 0) BSPMM_TRACE(p, 10);
      if (!VEC) {
        float* dst = reinterpret_cast<float*>(st);
        const int32_t total = n * kw;
        for (int32_t q = lane; q < total; q += 32) {
          const int32_t r = q / kw, c = q - r * kw;
          cp_async4(dst + q, bsrc + (int64_t)r * p.ldb + c);
        }
      }
      if (p.sbulk) {
        // <= 3 head and <= 3 tail elements per array, on lanes 24..31 (they
        // issue no TMA).  A branch-free variant on lanes 0..17 (addresses by
        // selects) measured slower on C5 (840 vs 810 us): lanes 0..2 have just
        // issued the slice's bulk copies
        if (lane >= 24 && lane < 27 && lane - 24 < a_col) {
          cp_async4(dcol + (lane - 24), p.col + nz0 + (lane - 24));
          cp_async4(dval + (lane - 24), p.vals + nz0 + (lane - 24));
        }
        if (lane >= 27 && lane < 30 && b_col + (lane - 27) < nnz) {
          cp_async4(dcol + b_col + (lane - 27), p.col + nz0 + b_col + (lane - 27));
          cp_async4(dval + b_col + (lane - 27), p.vals + nz0 + b_col + (lane - 27));
        }
        if (lane == 30)
          for (int32_t r = 0; r < a_rp; ++r) cp_async4(drp + r, p.row_ptr + r_lo + r);
        if (lane == 31)
          for (int32_t r = b_rp; r < r_cnt; ++r) cp_async4(drp + r, p.row_ptr + r_lo + r);
      } else {  // unaligned bases: the whole slice by 4-byte copies
        for (int32_t e = lane; e < nnz; e += 32) {
          cp_async4(dcol + e, p.col + nz0 + e);
          cp_async4(dval + e, p.vals + nz0 + e);
        }
        for (int32_t r = lane; r < r_cnt; r += 32) cp_async4(drp + r, p.row_ptr + r_lo + r);
      }
    }
    if (p.trace) __syncwarp();
    if (j < 3 && lane == 0) BSPMM_TRACE(p, 19 + 4 * j);
    if (lane == 0) {
      UnitHdr h;
      h.g0 = g0; h.n = n; h.nz0 = nz0; h.nnz = nnz; h.c0 = c0; h.kw = kw;
      h.flags = (bst ? 1 : 0) | (sst ? 2 : 0) | (b_early ? 8 : 0);
      hdr[s] = h;
      mbar_arrive(&full[s]);  // release: header visible to consumers
    }
    if (j < 2 && lane == 0) BSPMM_TRACE(p, 11 + j);
    cp_async_arrive_noinc(&full[s]);  // 32 arrivals, each after its lane's copies land
    if (j < 2 && lane == 0) BSPMM_TRACE(p, 13 + j);
}

// After the last unit: a "done" header (flags = -1) tells the consumers to exit.
__device__ __forceinline__ void issue_done(const SpmmParams& p, unsigned char* smem, int j) {
  UnitHdr* hdr = reinterpret_cast<UnitHdr*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * kHdrBytes);
  uint64_t* empty = full + p.stages;
  const int lane = threadIdx.x & 31;
  const int s = j % p.stages;
  mbar_wait(&empty[s], ((uint32_t)(j / p.stages) & 1u) ^ 1u);
  uint64_t* sfull = sfull_bar(p, smem);
  if (lane == 0) {
    hdr[s].flags = -1;
    if (p.nnz_off) mbar_arrive(&sfull[s]);
    mbar_arrive(&full[s]);
  }
  cp_async_arrive_noinc(p.nnz_off ? &sfull[s] : &full[s]);
}

template <bool VEC, bool COO>
__device__ __forceinline__ void produce(const SpmmParams& p, const TmaMaps& maps, unsigned char* smem) {
  const int lane = threadIdx.x & 31;
  const int64_t G = gridDim.x;
  int j = 0;
  // Static schedule (default): units blockIdx.x, +grid, ...  Metadata for 32
  // units per batch, one lane each, both round trips done BEFORE any copy of
  // the batch is issued: under load the row_ptr loads would otherwise queue
  // behind the bulk B traffic (tools/trace.py).  The next batch is prefetched
  // while the current one is issued.
  // Dynamic schedule (p.sched, mixed-size batches): the first unit is
  // blockIdx.x, later ones come from a global ticket counter, so a CTA that
  // drew small matrices keeps drawing (load balance within one unit).  The
  // next ticket is drawn while the current unit is issued.  The counter resets
  // itself: the draw that returns units - 1 is the last of the launch.
  // Both feed ONE issue_unit call site (instruction-cache footprint).
  Meta cur, nxt;
  int64_t carry = 0;
  unsigned long long t_next = 0;
  int64_t u = blockIdx.x;
  if (p.sched) {
    if (lane == 0) {
      t_next = atomicAdd(p.sched, 1ULL);
      meta_rt1<COO>(p, u, cur);
      meta_rt2<COO>(p, u, cur);
    }
  } else {
    carry = p.row_off ? 0 : fused_prefix_start(p, lane);
    meta_rt1<COO>(p, blockIdx.x + lane * G, nxt, p.row_off ? -1 : fused_prefix(p, blockIdx.x, G, lane, carry));
    meta_rt2<COO>(p, blockIdx.x + lane * G, nxt);
  }
  while (u < p.units) {
    int src = 0;  // lane holding this unit's metadata
    if (!p.sched) {
      const int jj = j & 31;
      if (jj == 0) {
        cur = nxt;
        const int64_t nb = u + 32 * G;  // next batch, round trip 1
        meta_rt1<COO>(p, nb + lane * G, nxt, p.row_off ? -1 : fused_prefix(p, nb, G, lane, carry));
        if (j == 0 && lane == 0) BSPMM_TRACE(p, 2);
      }
      if (jj == 8 || (jj == 0 && u + 8 * G >= p.units)) meta_rt2<COO>(p, u + (32 - jj + lane) * G, nxt);
      src = jj;
    }
    const int64_t g0 = __shfl_sync(0xffffffffu, cur.g0, src);
    const int32_t n = __shfl_sync(0xffffffffu, cur.n, src);
    const int32_t c0 = __shfl_sync(0xffffffffu, cur.c0, src);
    const int32_t kw = __shfl_sync(0xffffffffu, cur.kw, src);
    const int32_t nz0 = __shfl_sync(0xffffffffu, cur.nz0, src);
    const int32_t nnz = __shfl_sync(0xffffffffu, cur.nz1, src) - nz0;
    if (j == 0 && lane == 0) BSPMM_TRACE(p, 3);
    issue_unit<VEC, COO>(p, maps, smem, j, g0, n, c0, kw, nz0, nnz, j == 0 && early_b_ok<VEC, COO>(p, n, kw));
    ++j;
    if (p.sched) {
      const unsigned long long t = __shfl_sync(0xffffffffu, t_next, 0);
      if ((int64_t)t + G >= p.units) {
        if (lane == 0 && t == (unsigned long long)p.units - 1) atomicExch(p.sched, 0ULL);
        break;
      }
      u = (int64_t)t + G;
      if (lane == 0) {
        t_next = atomicAdd(p.sched, 1ULL);
        meta_rt1<COO>(p, u, cur);
        meta_rt2<COO>(p, u, cur);
      }
    } else {
      u += G;
    }
  }
  issue_done(p, smem, j);
  if (lane == 0) BSPMM_TRACE(p, 4);
}

// a-5/a-6 for one unit: a sub-warp of L lanes owns a row; each lane owns CH
// column chunks (float4 when VEC) at lane-strided positions li + v*L (the
// paper's j = lane, lane + subWarp, ..., in 128-bit chunks).  Up
// to G entries of a row are loaded ahead (independent shared-memory loads),
// then accumulated strictly in storage order, so the result is bitwise the
// fp32 storage-order FMA sum (O3').  Per-unit address math is hoisted; the
// row loop touches shared memory with 32-bit offsets only.
template <int CH, bool VEC, bool BST, bool SST, int EPI>
__device__ __forceinline__ void rows(const SpmmParams& p, const UnitHdr& h, const unsigned char* st, int first,
                                     int step, int li) {
  constexpr int G = CH >= 4 ? 2 : 4;
  constexpr int FW = VEC ? 4 : 1;  // floats per chunk
  const int L = p.lanes;
  const int32_t cols = VEC ? (h.kw >> 2) : h.kw;
  bool ok[CH];
#pragma unroll
  for (int v = 0; v < CH; ++v) ok[v] = li + v * L < cols;
  // row pointers, column ids and values of the slice, indexed by ABSOLUTE entry position
  const unsigned char* sreg = st + p.stage_b;
  const int32_t* rp = SST ? reinterpret_cast<const int32_t*>(sreg + 2 * slice_region(h.nnz)) + (h.g0 & 3)
                          : p.row_ptr + h.g0;
  const int32_t* col_i = SST ? reinterpret_cast<const int32_t*>(sreg) + (h.nz0 & 3) - h.nz0 : p.col;
  const float* col_v = SST ? reinterpret_cast<const float*>(sreg + slice_region(h.nnz)) + (h.nz0 & 3) - h.nz0 : p.vals;
  // B rows of the tile (lane offset folded in) and C rows
  const float* Bt = BST ? reinterpret_cast<const float*>(st) + FW * li : p.B + h.g0 * p.ldb + h.c0 + FW * li;
  const int64_t bstride = BST ? (int64_t)h.kw : p.ldb;
  float* Ct = p.C + h.g0 * p.ldc + h.c0 + FW * li;
  int r = first;
  int32_t nx0 = 0, nx1 = 0;
  if (r < h.n) {
    nx0 = rp[r];
    nx1 = rp[r + 1];
  }
  for (; r < h.n; r += step) {
    const int32_t e0 = nx0, e1 = nx1;
    if (r + step < h.n) {  // next row's range, loaded ahead
      nx0 = rp[r + step];
      nx1 = rp[r + step + 1];
    }
    float4 acc[CH];
#pragma unroll
    for (int v = 0; v < CH; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    float rs = 0.f;  // row sum of A (GCN bias epilogue)
    for (int32_t e = e0; e < e1; e += G) {
      const int32_t cnt = min(G, e1 - e);
      int32_t cidx[G];
      float a[G];
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (q < cnt) {
          if (SST) {
            cidx[q] = col_i[e + q];
            a[q] = col_v[e + q];
          } else {
            cidx[q] = __ldg(col_i + e + q);
            a[q] = __ldg(col_v + e + q);
          }
        }
      }
      float4 b[G][CH];
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (q < cnt) {
          const float* brow = BST ? Bt + (int32_t)(cidx[q] * (int32_t)bstride) : Bt + (int64_t)cidx[q] * bstride;
#pragma unroll
          for (int v = 0; v < CH; ++v) {
            if (ok[v]) {
              if (VEC) b[q][v] = BST ? *reinterpret_cast<const float4*>(brow + FW * v * L) : ldg_nc_f4(brow + FW * v * L);
              else b[q][v].x = BST ? brow[v * L] : __ldg(brow + v * L);
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (q < cnt) {
          if (EPI == 1) rs += a[q];
#pragma unroll
          for (int v = 0; v < CH; ++v) {
            acc[v].x = fmaf(a[q], b[q][v].x, acc[v].x);
            if (VEC) {
              acc[v].y = fmaf(a[q], b[q][v].y, acc[v].y);
              acc[v].z = fmaf(a[q], b[q][v].z, acc[v].z);
              acc[v].w = fmaf(a[q], b[q][v].w, acc[v].w);
            }
          }
        }
      }
    }
    float* crow = Ct + (int64_t)r * p.ldc;
    if (p.dbg & 1) {
      if (acc[0].x == 1.2345e-38f) crow[0] = 0.f;  // keep the math alive, store nothing
      continue;
    }
#pragma unroll
    for (int v = 0; v < CH; ++v) {
      if (ok[v]) {
        epilogue<EPI, VEC>(p, acc[v], rs, h.c0 + FW * (li + v * L), crow + FW * v * L);
        store_c<EPI, VEC>(p, crow + FW * v * L, acc[v]);
      }
    }
  }
}

// units that did not fit a stage (the paper's case 3): the
// same storage-order sum read straight from global memory (L1/L2-cached B
// gathers), a plain loop to keep the register allocation of the staged path
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void fma4(float4& acc, float a, const float4& b) {
  acc.x = fmaf(a, b.x, acc.x);
  acc.y = fmaf(a, b.y, acc.y);
  acc.z = fmaf(a, b.z, acc.z);
  acc.w = fmaf(a, b.w, acc.w);
}

// The hot loop for a staged unit whose tile is covered exactly by the lanes
// (cols == lanes * CH, float4 chunks): no per-chunk predicates, 32-bit shared
// addressing, two entries per iteration (independent loads first, FMAs in
// storage order).  Same arithmetic as rows<> (bitwise O3').
template <int CH, int EPI>
__device__ __forceinline__ void rows_staged_full(const SpmmParams& p, const UnitHdr& h, const unsigned char* st,
                                                 int first, int step, int li) {
  const int L = p.lanes;
  const uint32_t pitch = (uint32_t)h.kw * 4u;
  const uint32_t sB = smem_addr(st) + 16u * (uint32_t)li;
  const uint32_t vstep = 16u * (uint32_t)L;
  const unsigned char* sreg = st + p.stage_b;
  const int32_t* rp = reinterpret_cast<const int32_t*>(sreg + 2 * slice_region(h.nnz)) + (h.g0 & 3);
  const int32_t* ci = reinterpret_cast<const int32_t*>(sreg) + (h.nz0 & 3) - h.nz0;
  const float* cv = reinterpret_cast<const float*>(sreg + slice_region(h.nnz)) + (h.nz0 & 3) - h.nz0;
  float* Ct = p.C + h.g0 * p.ldc + h.c0 + 4 * li;
  int r = first;
  int32_t nx0 = 0, nx1 = 0;
  if (r < h.n) {
    nx0 = rp[r];
    nx1 = rp[r + 1];
  }
  for (; r < h.n; r += step) {
    int32_t e = nx0;
    const int32_t e1 = nx1;
    if (r + step < h.n) {
      nx0 = rp[r + step];
      nx1 = rp[r + step + 1];
    }
    float4 acc[CH];
#pragma unroll
    for (int v = 0; v < CH; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    float rs = 0.f;  // row sum of A (GCN bias epilogue)
    for (; e + 1 < e1; e += 2) {
      const int32_t c0 = ci[e], c1 = ci[e + 1];
      const float a0 = cv[e], a1 = cv[e + 1];
      const uint32_t p0 = sB + (uint32_t)c0 * pitch, p1 = sB + (uint32_t)c1 * pitch;
      float4 x0[CH], x1[CH];
#pragma unroll
      for (int v = 0; v < CH; ++v) {
        x0[v] = lds128(p0 + v * vstep);
        x1[v] = lds128(p1 + v * vstep);
      }
#pragma unroll
      for (int v = 0; v < CH; ++v) fma4(acc[v], a0, x0[v]);
#pragma unroll
      for (int v = 0; v < CH; ++v) fma4(acc[v], a1, x1[v]);
      if (EPI == 1) rs += a0, rs += a1;
    }
    if (e < e1) {
      const int32_t c0 = ci[e];
      const float a0 = cv[e];
      if (EPI == 1) rs += a0;
      const uint32_t p0 = sB + (uint32_t)c0 * pitch;
#pragma unroll
      for (int v = 0; v < CH; ++v) fma4(acc[v], a0, lds128(p0 + v * vstep));
    }
    float* crow = Ct + (int64_t)r * p.ldc;
    if (p.dbg & 1) {
      if (acc[0].x == 1.2345e-38f) crow[0] = 0.f;  // keep the math alive, store nothing
      continue;
    }
#pragma unroll
    for (int v = 0; v < CH; ++v) {
      epilogue<EPI, true>(p, acc[v], rs, h.c0 + 4 * (li + v * L), crow + 4 * v * L);
      store_c<EPI, true>(p, crow + 4 * v * L, acc[v]);
    }
  }
}

// SDDMM rows (EPI == 3): the same sub-warp row ownership and staged B_i as
// the SpMM, but each entry's result is a dot product: lane li holds its float4
// chunks of the row's grad_C (loaded one row ahead from global memory), forms
// its partial <G[r], B[col_e]> over them (fixed order), and the L lanes of the
// sub-warp reduce it with a fixed xor butterfly (deterministic; within the
// north_star bound of the fp64 oracle O6).  BST: B tile and CSR slice staged.
// Used for latency-bound batches only: on streaming batches the per-row
// grad_C loads leave too few bytes in flight per SM (C5 1200 us vs 1071 us
// for the standalone kernel; a two-row register double buffer measured
// slower, 1525 us, no-allocate loads changed nothing, and warp-uniform loops
// with full-mask shuffles for sub-warp rows were slower on every config).
template <int CH, bool BST>
__device__ __forceinline__ void rows_sddmm(const SpmmParams& p, const UnitHdr& h, const unsigned char* st, int first,
                                           int step, int li, int sub) {
  const int L = p.lanes;
  const int32_t cols = h.kw >> 2;
  bool ok[CH];
#pragma unroll
  for (int v = 0; v < CH; ++v) ok[v] = li + v * L < cols;
  const unsigned char* sreg = st + p.stage_b;
  const int32_t* rp = BST ? reinterpret_cast<const int32_t*>(sreg + 2 * slice_region(h.nnz)) + (h.g0 & 3)
                          : p.row_ptr + h.g0;
  const int32_t* ci = BST ? reinterpret_cast<const int32_t*>(sreg) + (h.nz0 & 3) - h.nz0 : p.col;
  const float* Bt = BST ? reinterpret_cast<const float*>(st) + 4 * li : p.B + h.g0 * p.ldb + h.c0 + 4 * li;
  const int64_t bstride = BST ? (int64_t)h.kw : p.ldb;
  const float* Gt = p.G + h.g0 * p.ldg + h.c0 + 4 * li;
  const uint32_t mask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (sub * L));
  auto gload = [&](int r_, float4* dst) {
    const float* g = Gt + (int64_t)r_ * p.ldg;
#pragma unroll
    for (int v = 0; v < CH; ++v)  // read once: no L1 allocation (C4 10.1 -> 9.5 us)
      dst[v] = ok[v] ? ldg_na_f4(g + 4 * v * L) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  auto bload = [&](int32_t c, int v) -> float4 {
    const float* b = Bt + (int64_t)c * bstride + 4 * v * L;
    return BST ? *reinterpret_cast<const float4*>(b) : ldg_nc_f4(b);
  };
  // all lanes of a sub-warp reduce q over the sub-warp (fixed xor butterfly)
  auto reduce = [&](float q) {
    if (L == 32) {  // whole-warp rows: a constant mask, no convergence checks per shuffle (C4 9.5 -> 8.0 us)
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) q += __shfl_xor_sync(0xffffffffu, q, d);
    } else {
      for (int d = L >> 1; d > 0; d >>= 1) q += __shfl_xor_sync(mask, q, d);
    }
    return q;
  };
  // two reductions interleaved (independent shuffle chains)
  auto reduce2 = [&](float& q0, float& q1) {
    if (L == 32) {
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        q0 += __shfl_xor_sync(0xffffffffu, q0, d);
        q1 += __shfl_xor_sync(0xffffffffu, q1, d);
      }
    } else {
      for (int d = L >> 1; d > 0; d >>= 1) {
        q0 += __shfl_xor_sync(mask, q0, d);
        q1 += __shfl_xor_sync(mask, q1, d);
      }
    }
  };
  auto dot = [&](const float4* g, const float4* b) {
    float q = 0.f;
#pragma unroll
    for (int v = 0; v < CH; ++v) {
      q = fmaf(g[v].x, b[v].x, q);
      q = fmaf(g[v].y, b[v].y, q);
      q = fmaf(g[v].z, b[v].z, q);
      q = fmaf(g[v].w, b[v].w, q);
    }
    return q;
  };
  int r = first;
  int32_t nx0 = 0, nx1 = 0;
  float4 gn[CH];
  if (r < h.n) {
    nx0 = rp[r];
    nx1 = rp[r + 1];
    gload(r, gn);
  }
  for (; r < h.n; r += step) {
    const int32_t e1 = nx1;
    int32_t e = nx0;
    float4 gv[CH];
#pragma unroll
    for (int v = 0; v < CH; ++v) gv[v] = gn[v];
    if (r + step < h.n) {  // next row's range and grad_C chunks, loaded ahead
      nx0 = rp[r + step];
      nx1 = rp[r + step + 1];
      gload(r + step, gn);
    }
    for (; e + 1 < e1; e += 2) {
      const int32_t c0 = ci[e], c1 = ci[e + 1];
      float4 b0[CH], b1[CH];
#pragma unroll
      for (int v = 0; v < CH; ++v) {
        b0[v] = ok[v] ? bload(c0, v) : make_float4(0.f, 0.f, 0.f, 0.f);
        b1[v] = ok[v] ? bload(c1, v) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      float q0 = dot(gv, b0), q1 = dot(gv, b1);
      reduce2(q0, q1);
      if (li == 0) {
        p.sd_out[e] = q0;
        p.sd_out[e + 1] = q1;
      }
    }
    if (e < e1) {
      const int32_t c0 = ci[e];
      float4 b0[CH];
#pragma unroll
      for (int v = 0; v < CH; ++v) b0[v] = ok[v] ? bload(c0, v) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float q0 = reduce(dot(gv, b0));
      if (li == 0) p.sd_out[e] = q0;
    }
  }
}

template <int CH, bool VEC, int EPI>
__device__ __forceinline__ void rows_direct(const SpmmParams& p, const UnitHdr& h, int first, int step, int li) {
  constexpr int FW = VEC ? 4 : 1;
  const int L = p.lanes;
  const int32_t cols = VEC ? (h.kw >> 2) : h.kw;
  const int32_t* rp = p.row_ptr + h.g0;
  const float* Bt = p.B + h.g0 * p.ldb + h.c0 + FW * li;
  float* Ct = p.C + h.g0 * p.ldc + h.c0 + FW * li;
  for (int r = first; r < h.n; r += step) {
    const int32_t e0 = __ldg(rp + r), e1 = __ldg(rp + r + 1);
    float4 acc[CH];
#pragma unroll
    for (int v = 0; v < CH; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    float rs = 0.f;
    for (int32_t e = e0; e < e1; ++e) {
      const int32_t c = __ldg(p.col + e);
      const float a = __ldg(p.vals + e);
      if (EPI == 1) rs += a;
      const float* brow = Bt + (int64_t)c * p.ldb;
#pragma unroll
      for (int v = 0; v < CH; ++v) {
        if (li + v * L < cols) {
          if (VEC) {
            const float4 b = ldg_nc_f4(brow + FW * v * L);
            acc[v].x = fmaf(a, b.x, acc[v].x);
            acc[v].y = fmaf(a, b.y, acc[v].y);
            acc[v].z = fmaf(a, b.z, acc[v].z);
            acc[v].w = fmaf(a, b.w, acc[v].w);
          } else {
            acc[v].x = fmaf(a, __ldg(brow + v * L), acc[v].x);
          }
        }
      }
    }
    float* crow = Ct + (int64_t)r * p.ldc;
#pragma unroll
    for (int v = 0; v < CH; ++v) {
      if (li + v * L < cols) {
        epilogue<EPI, VEC>(p, acc[v], rs, h.c0 + FW * (li + v * L), crow + FW * v * L);
        store_c<EPI, VEC>(p, crow + FW * v * L, acc[v]);
      }
    }
  }
}

// Fused COO -> CSR of one staged unit (row a-2 inside the SpMM): counting
// sort by row + rank of the unique key (col, original position) within each
// row segment -- the same canonical order as coo2csr.cu, so the SpMM that
// follows is bitwise identical to the two-kernel path.  Converter warps only
// (named barrier 2); writes the standard CSR slice layout of the stage.
// (named barrier 2: the converter warps)
__device__ __forceinline__ void consumer_bar(int T) { asm volatile("bar.sync 2, %0;" ::"r"(T) : "memory"); }

__device__ __forceinline__ void coo_convert(const SpmmParams& p, const UnitHdr& h, unsigned char* st, int t, int T,
                                            bool tr) {
  unsigned char* sreg = st + p.stage_b;
  const int32_t nnz = h.nnz, n = h.n, z0 = h.nz0;
  unsigned char* raw = sreg + coo_raw_off(nnz, n);
  const int2* pr = reinterpret_cast<const int2*>(raw) + (z0 & 1);
  const float* rv = reinterpret_cast<const float*>(raw + coo_pairs_bytes(nnz)) + (z0 & 3);
  int32_t* slot = reinterpret_cast<int32_t*>(raw + coo_pairs_bytes(nnz) + coo_vals_bytes(nnz));
  int32_t* cursor = reinterpret_cast<int32_t*>(sreg + p.stage_s - coo_cursor_bytes(p.coo_rows));  // zero here
  int32_t* col = reinterpret_cast<int32_t*>(sreg) + (z0 & 3);
  float* val = reinterpret_cast<float*>(sreg + slice_region(nnz)) + (z0 & 3);
  int32_t* rp = reinterpret_cast<int32_t*>(sreg + 2 * slice_region(nnz)) + (h.g0 & 3);
  for (int32_t e = t; e < nnz; e += T) atomicAdd(&cursor[pr[e].x], 1);
  consumer_bar(T);
  if (tr && t == 0) BSPMM_TRACE(p, 28);
  // exclusive scan of the row counts into the row pointers, one phase: the
  // warp that owns a 32-row chunk sums the counts of every row before it
  // itself (no chunk-total exchange, no second barrier); the counts stay in
  // `cursor` for the scatter
  const int32_t nchunk = (n + 31) >> 5;
  const int lt = t & 31;
  for (int32_t c = t >> 5; c < nchunk; c += T >> 5) {
    int32_t base = 0;
    for (int32_t q = lt; q < 32 * c; q += 32) base += cursor[q];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) base += __shfl_xor_sync(0xffffffffu, base, d);
    const int32_t r = c * 32 + lt;
    const int32_t v = r < n ? cursor[r] : 0;
    int32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lt >= d) x += y;
    }
    if (r < n) rp[r] = z0 + base + x - v;
  }
  if (t == 0) rp[n] = z0 + nnz;
  consumer_bar(T);
  if (tr && t == 0) BSPMM_TRACE(p, 29);
  // scatter into the row segments (any order within a segment: sorted next);
  // the count is consumed downwards
  for (int32_t e = t; e < nnz; e += T) {
    const int32_t r = pr[e].x;
    slot[rp[r] - z0 + atomicSub(&cursor[r], 1) - 1] = e;
  }
  consumer_bar(T);
  if (tr && t == 0) BSPMM_TRACE(p, 30);
  // order within each row segment by the unique key (col, original position):
  // a thread per row sorts up to 8 keys in registers (a sorting network; the
  // molecule and paper-style graphs have <= 8 entries per row), longer rows
  // rank each entry by counting smaller keys in its segment
  for (int32_t r = t; r < n; r += T) {
    const int32_t s0 = rp[r] - z0, s1 = rp[r + 1] - z0, d = s1 - s0;
    if (d <= 8) {
      // key = (col << 16) | position: unique, ordered as (col, position); both
      // fit 16 bits (a stage holds < 2^16 rows and entries)
      uint32_t key[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int32_t e = q < d ? slot[s0 + q] : 0;
        key[q] = q < d ? ((uint32_t)pr[e].y << 16) | (uint32_t)e : 0xffffffffu;
      }
#define BSPMM_CX(a, b)                                   \
      {                                                  \
        const uint32_t lo = min(key[a], key[b]);         \
        key[b] = max(key[a], key[b]);                    \
        key[a] = lo;                                     \
      }
      if (d <= 4) {  // 4 keys: 5 compare-exchanges
        BSPMM_CX(0, 1) BSPMM_CX(2, 3) BSPMM_CX(0, 2) BSPMM_CX(1, 3) BSPMM_CX(1, 2)
      } else {       // Batcher's odd-even merge sort network, 8 keys (19)
        BSPMM_CX(0, 1) BSPMM_CX(2, 3) BSPMM_CX(4, 5) BSPMM_CX(6, 7)
        BSPMM_CX(0, 2) BSPMM_CX(1, 3) BSPMM_CX(4, 6) BSPMM_CX(5, 7)
        BSPMM_CX(1, 2) BSPMM_CX(5, 6)
        BSPMM_CX(0, 4) BSPMM_CX(1, 5) BSPMM_CX(2, 6) BSPMM_CX(3, 7)
        BSPMM_CX(2, 4) BSPMM_CX(3, 5)
        BSPMM_CX(1, 2) BSPMM_CX(3, 4) BSPMM_CX(5, 6)
      }
#undef BSPMM_CX
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (q < d) {
          const int32_t e = (int32_t)(key[q] & 0xffffu);
          col[s0 + q] = (int32_t)(key[q] >> 16);
          val[s0 + q] = rv[e];  // bitwise move
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
        col[s0 + rank] = ce;
        val[s0 + rank] = rv[e];
      }
    }
  }
  consumer_bar(T);
  if (tr && t == 0) BSPMM_TRACE(p, 31);
}

template <int CH, bool VEC, int EPI, bool COO, bool ONE>
__device__ __forceinline__ void consume(const SpmmParams& p, const TmaMaps& maps, unsigned char* smem) {
  const UnitHdr* hdr = reinterpret_cast<const UnitHdr*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * kHdrBytes);
  uint64_t* empty = full + p.stages;
  const unsigned char* ring = smem + ring_prefix_bytes(p.stages);
  const int32_t stage_bytes = p.stage_b + p.stage_s;
  const int lane = threadIdx.x & 31;
  const int cw = (threadIdx.x >> 5) - 1;
  const int W = (blockDim.x >> 5) - 1 - (COO ? p.cvt_warps : 0);
  const int L = p.lanes;
  const int rpw = 32 / L;
  const int sub = lane / L, li = lane % L;
  const int first = cw * rpw + sub, step = W * rpw;
  if (VEC && !COO && cw == 0 && !p.sched && !(p.dbg & (2 | 4)))
    early_b_issue(p.row_off, p.sizes, p.B, p.ldb, p.tiles, p.kt, p.k, p.stage_b, p.trace,
                  early_bar(p, const_cast<unsigned char*>(smem)), const_cast<unsigned char*>(ring));
  int j0 = 0;
  if (ONE) {
    // one whole-row unit per CTA whose rows the consumer warps cover in one
    // round (small latency-bound batches, e.g. C2): the consumers do not wait
    // for the producer's header and CSR slice -- every warp loads the unit's
    // row range itself, waits only for the early B tile and reads its rows'
    // structure from global memory (those loads overlap the B landing; the
    // producer's slice path is the critical path otherwise, trace).  The
    // producer still stages unit 0 as usual: its copies are waited for
    // (full[0], phase 0) BEFORE arriving on empty[0] -- the producer cannot
    // advance full[0] past phase 0 until every warp has arrived.
    const int64_t i = blockIdx.x;
    const int32_t ni = p.sizes ? __ldg(p.sizes + i) : 0;
    const int64_t g0 = p.row_off ? p.row_off[i] : warp_sizes_sum(p.sizes, i, lane);
    const int32_t n = p.sizes ? ni : (int32_t)(p.row_off[i + 1] - g0);
    const int32_t kw = min(p.kt, p.k);  // as the producer and early_b_issue compute it
    if (n <= step && early_b_ok<VEC, COO>(p, n, kw)) {
      UnitHdr h;
      h.g0 = g0; h.n = n; h.nz0 = 0; h.nnz = 0; h.c0 = 0; h.kw = kw; h.flags = 1;
      mbar_wait(early_bar(p, const_cast<unsigned char*>(smem)), 0u);
      if (cw == 0 && lane == 0) BSPMM_TRACE(p, 5);
      rows<CH, VEC, true, false, EPI>(p, h, ring, first, step, li);
      mbar_wait(&full[0], 0u);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[0]);
      if (cw == 0 && lane == 0) BSPMM_TRACE(p, 8);
      j0 = 1;
    }
  }
  for (int j = j0;; ++j) {
    const int s = j % p.stages;
    const uint32_t par = (uint32_t)(j / p.stages) & 1u;
    // fused COO mode: the slice (and header) first; its conversion overlaps
    // the B tile's landing, waited for below
    mbar_wait(COO ? &sfull_bar(p, const_cast<unsigned char*>(smem))[s] : &full[s], par);
    if (j == 0 && cw == 0 && lane == 0) BSPMM_TRACE(p, 5);
    const UnitHdr h = hdr[s];
    if (h.flags < 0) break;  // the producer's "done" header
    if (j == 0 && (h.flags & 8)) mbar_wait(early_bar(p, const_cast<unsigned char*>(smem)), 0u);  // early B tile
    const unsigned char* st = ring + (size_t)s * stage_bytes;
    if (COO) {  // the converter warps' CSR slice, then the B tile
      mbar_wait(&cvt_bar(p, const_cast<unsigned char*>(smem))[s], par);
      mbar_wait(&full[s], par);
    }
    const int reps = (p.dbg & 8) ? 4 : 1;  // debug: repeat the unit's work (consumer cost in isolation)
    for (int rep = 0; rep < reps && (h.flags & 4) == 0; ++rep) {  // 4: COO unit over capacity (skipped, flagged)
      if (EPI == 3) {  // SDDMM mode (NEXT-2)
        if ((h.flags & 3) == 3) rows_sddmm<CH, true>(p, h, st, first, step, li, sub);
        else rows_sddmm<CH, false>(p, h, st, first, step, li, sub);
      } else if ((h.flags & 3) == 3) {  // the hot, staged case
        if (VEC && (h.kw >> 2) == p.lanes * CH) rows_staged_full<CH, EPI>(p, h, st, first, step, li);
        else rows<CH, VEC, true, true, EPI>(p, h, st, first, step, li);
      } else {
        rows_direct<CH, VEC, EPI>(p, h, first, step, li);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (j == 0 && cw == 0 && lane == 0) BSPMM_TRACE(p, 8);
  }
  // multicast stores: make them visible system-wide before the caller's
  // cross-GPU barrier (which follows this kernel on the stream)
  if (EPI == 2) __threadfence_system();
  if (cw == 0 && lane == 0) BSPMM_TRACE(p, 6);
}

// Fused COO mode: the converter warps walk the units in the consumers' order.
// Unit j's SparseTensor slice is converted as soon as it lands (sfull), while
// the consumer warps still compute unit j-1 -- the conversion leaves the
// consumers' critical path except for a CTA's first unit.  Every unit's
// "converted" barrier is arrived on (also units that need no conversion), so
// its phases stay in step with the ring.
__device__ __forceinline__ void convert_units(const SpmmParams& p, unsigned char* smem, int W) {
  const UnitHdr* hdr = reinterpret_cast<const UnitHdr*>(smem);
  unsigned char* ring = smem + ring_prefix_bytes(p.stages);
  const int32_t stage_bytes = p.stage_b + p.stage_s;
  const int t = threadIdx.x - 32 * (1 + W);
  for (int j = 0;; ++j) {
    const int s = j % p.stages;
    const uint32_t par = (uint32_t)(j / p.stages) & 1u;
    mbar_wait(&sfull_bar(p, smem)[s], par);
    const UnitHdr h = hdr[s];
    if (h.flags < 0) break;  // the producer's "done" header
    if ((h.flags & 3) == 3)  // SparseTensor slice -> CSR slice in shared memory
      coo_convert(p, h, ring + (size_t)s * stage_bytes, t, p.cvt_warps * 32, j == 0);
    __syncwarp();
    if ((t & 31) == 0) mbar_arrive(&cvt_bar(p, smem)[s]);
  }
}

// Pre-wait prologue (programmatic dependent launch), batches with at most 8
// units per CTA: consumer warp 0 (idle until the first unit lands) prefetches
// into L2, BEFORE griddepcontrol.wait, the B rows and the structure slice of
// this CTA's units -- a CTA becomes resident as soon as the previous launch's
// CTA on its SM exits, so the prefetch fills the previous launch's tail (C3:
// its CTAs finish over a ~5 us spread).  The row and entry ranges are read
// with relaxed loads that may race with the previous kernel; the prefetches
// are hints clipped to the arrays' allocations, and everything the kernel
// uses is read again after the wait.
template <bool COO>
__device__ __forceinline__ void prefetch_units(const SpmmParams& p) {
  const int lane = threadIdx.x & 31;
  const int64_t u = blockIdx.x + (int64_t)lane * gridDim.x;
  if (lane >= 8 || u >= p.units) return;
  const int64_t i = u / p.tiles;
  if (u - i * p.tiles != 0 && u != blockIdx.x) return;  // a matrix's rows once per CTA
  const int64_t g0 = ld_relaxed_s64(p.row_off + i);
  const int64_t g1 = p.sizes ? g0 + ld_relaxed_s32(p.sizes + i) : ld_relaxed_s64(p.row_off + i + 1);
  if (g1 <= g0 || g1 - g0 > (1 << 20)) return;
  prefetch_l2_clipped(reinterpret_cast<uint64_t>(p.B + g0 * p.ldb), (uint64_t)(g1 - g0) * p.ldb * 4, p.b_lo,
                      p.b_hi);
  if (p.g_hi)  // SDDMM mode: the grad_C rows the consumers read from global memory
    prefetch_l2_clipped(reinterpret_cast<uint64_t>(p.G + g0 * p.ldg), (uint64_t)(g1 - g0) * p.ldg * 4, p.g_lo,
                        p.g_hi);
  if (COO) {
    if (!p.s_hi[1]) return;
    const int64_t z0 = ld_relaxed_s64(p.nnz_off + i), z1 = ld_relaxed_s64(p.nnz_off + i + 1);
    if (z1 <= z0 || z1 - z0 > (1 << 24)) return;
    prefetch_l2_clipped(reinterpret_cast<uint64_t>(p.idx + 2 * z0), (uint64_t)(z1 - z0) * 8, p.s_lo[1], p.s_hi[1]);
    prefetch_l2_clipped(reinterpret_cast<uint64_t>(p.vals + z0), (uint64_t)(z1 - z0) * 4, p.s_lo[2], p.s_hi[2]);
  } else if (p.s_hi[0]) {
    prefetch_l2_clipped(reinterpret_cast<uint64_t>(p.row_ptr + g0), (uint64_t)(g1 - g0 + 1) * 4, p.s_lo[0],
                        p.s_hi[0]);
  }
}

template <int CH, bool VEC, int EPI, bool COO, bool ONE = false>
__global__ void __launch_bounds__(kMaxThreadsK(CH, COO), 1) __maxnreg__(kMaxRegsK(CH, COO)) spmm_csr_kernel(const SpmmParams p, const __grid_constant__ TmaMaps maps) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * kHdrBytes);
  uint64_t* empty = full + p.stages;
  if (threadIdx.x == 0) BSPMM_TRACE(p, 0);
  if (threadIdx.x == 0) {
    const uint32_t W = (blockDim.x >> 5) - 1 - (COO ? p.cvt_warps : 0);
    for (int s = 0; s < p.stages; ++s) {
      // producer lane-0 arrive + 32 cp.async arrivals; fused COO mode: the
      // cp.async arrivals go to the slice barrier, full[s] tracks the B tile
      mbar_init(&full[s], COO ? 1 : 1 + 32);
      if (COO) mbar_init(&sfull_bar(p, smem)[s], 1 + 32);
      if (COO) mbar_init(&cvt_bar(p, smem)[s], p.cvt_warps);
      mbar_init(&empty[s], W);      // one arrival per consumer warp
    }
    mbar_init(early_bar(p, smem), 1);  // the first unit's early B tile
    fence_mbar_init();
  }
  if (COO) {  // the per-row counters of every stage start at zero (coo_cursor_bytes)
    unsigned char* ring = smem + ring_prefix_bytes(p.stages);
    const int32_t stage_bytes = p.stage_b + p.stage_s;
    const int32_t nc = (int32_t)(coo_cursor_bytes(p.coo_rows) / 4);
    for (int s = 0; s < p.stages; ++s) {
      int32_t* cur = reinterpret_cast<int32_t*>(ring + (size_t)s * stage_bytes + p.stage_b + p.stage_s) - nc;
      for (int32_t r = threadIdx.x; r < nc; r += blockDim.x) cur[r] = 0;
    }
  }
  __syncthreads();
  if (p.b_hi && p.row_off && (threadIdx.x >> 5) == 1) prefetch_units<COO>(p);
  // programmatic dependent launch: everything above overlapped the previous
  // kernel (e.g. the offsets builder); global memory is read only after this
  // (the prefetch hints aside)
  pdl_wait();
  pdl_launch_dependents();
  if (threadIdx.x == 0) BSPMM_TRACE(p, 1);
  const int Wc = (blockDim.x >> 5) - 1 - (COO ? p.cvt_warps : 0);
  if ((threadIdx.x >> 5) == 0) produce<VEC, COO>(p, maps, smem);
  else if (!COO || (int)(threadIdx.x >> 5) <= Wc) consume<CH, VEC, EPI, COO, ONE>(p, maps, smem);
  else convert_units(p, smem, Wc);
  if (p.trace) {
    __syncthreads();
    if (threadIdx.x == 0) BSPMM_TRACE(p, 7);
  }
}

template <int CH, bool VEC, int EPI, bool COO = false, bool ONE = false>
static cudaError_t launch_t(const SpmmParams& sp, const TmaMaps& maps, const bspmm_plan_t& plan, cudaStream_t s) {
  auto kern = spmm_csr_kernel<CH, VEC, EPI, COO, ONE>;
  static thread_local int configured_bytes[64] = {};  // per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (plan.smem_bytes > 47 * 1024 && configured_bytes[dev & 63] < plan.smem_bytes) {  // dynamic + static above 48 KB
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, plan.smem_bytes);
    if (e != cudaSuccess) return e;
    configured_bytes[dev & 63] = plan.smem_bytes;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(plan.grid);
  cfg.blockDim = dim3(plan.threads);
  cfg.dynamicSmemBytes = plan.smem_bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, sp, maps);
}

template <int CH, bool VEC>
static cudaError_t launch_e(int epi, const SpmmParams& sp, const TmaMaps& maps, const bspmm_plan_t& plan,
                            cudaStream_t s) {
  // fused COO mode (row a-2 inside the launch) is planned only for the vector
  // path with the plain epilogue: its own instantiation, so the CSR kernels
  // carry none of its code (instruction-cache footprint of latency-bound launches)
  if (sp.nnz_off) {
    if constexpr (VEC) {
      if (epi == 0) return launch_t<CH, VEC, 0, true>(sp, maps, plan, s);
    }
    return cudaErrorInvalidValue;
  }
  if constexpr (VEC) {
    if (epi == 3) return launch_t<CH, VEC, 3>(sp, maps, plan, s);
    // one whole-row unit per CTA, rows covered in one consumer round (decided
    // per CTA on the device): the consumers start without the producer's
    // header and slice (an instantiation of its own; plain and GCN epilogues)
    const int32_t rows_per_round = ((plan.threads >> 5) - 1) * (32 / plan.lanes);
    if (epi == 0 && plan.units <= plan.grid && plan.tiles == 1 && !sp.sched && plan.max_rows <= rows_per_round &&
        !(sp.dbg & (2 | 4 | 1024)))
      return launch_t<CH, VEC, 0, false, true>(sp, maps, plan, s);
  }
  if (epi == 2) return launch_t<CH, VEC, 2>(sp, maps, plan, s);
  // EPI 1 (the round-1 GCN bias / channel-accumulate epilogue) is no longer
  // instantiated: the GCN layer runs in gcn_fused.cu
  if (epi == 1) return cudaErrorInvalidValue;
  return launch_t<CH, VEC, 0>(sp, maps, plan, s);
}

cudaError_t launch_spmm_csr(const CsrArgs& a, const bspmm_plan_t& plan, cudaStream_t s) {
  if (plan.units == 0 || plan.grid == 0) return cudaSuccess;
  SpmmParams sp;
  sp.units = plan.units;
  sp.tiles = plan.tiles;
  sp.kt = plan.kt;
  sp.k = a.k;
  sp.stages = plan.stages;
  sp.stage_b = plan.stage_b_bytes;
  sp.stage_s = plan.stage_s_bytes;
  sp.lanes = plan.lanes;
  sp.row_off = a.row_off;
  sp.sizes = a.sizes;
  sp.row_ptr = a.row_ptr;
  sp.col = a.col;
  sp.vals = a.vals;
  sp.B = a.B;
  sp.ldb = a.ldb;
  sp.C = a.C;
  sp.ldc = a.ldc;
  sp.trace = a.trace;
  sp.dbg = a.dbg;
  sp.tma2d = a.maps != nullptr ? 1 : 0;
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
  sp.sbulk = (al16(a.col) && al16(a.vals) && al16(a.row_ptr)) ? 1 : 0;
  sp.slice_lsu = (plan.units <= 32LL * plan.grid && !(a.dbg & 32)) ? 1 : 0;
  sp.bias = a.bias;
  sp.accumulate = a.accumulate;
  sp.mc = a.mc;
  sp.G = a.G;
  sp.ldg = a.ldg;
  sp.sd_out = a.sd_out;
  // epilogue variant: 0 plain store, 1 GCN (bias / accumulate), 2 multicast store, 3 SDDMM
  const int epi = a.sd_out ? 3 : a.mc ? 2 : (a.bias != nullptr || a.accumulate != 0) ? 1 : 0;
  if (epi == 3 && (!plan.vec || plan.tiles != 1)) return cudaErrorInvalidValue;
  sp.sched = a.sched;
  sp.nnz_off = a.coo_nnz_off;
  sp.idx = a.coo_idx;
  sp.err = a.err;  // C4: 8.4 vs 9.0 us; C5: 835 vs 849
  sp.cvt_warps = a.cvt_warps;
  sp.coo_rows = plan.max_rows;
  const bool pf = plan.units <= 8LL * plan.grid && (epi != 3 || a.g_hi);
  sp.b_lo = pf ? a.b_lo : 0;
  sp.b_hi = pf ? a.b_hi : 0;
  sp.g_lo = pf && epi == 3 ? a.g_lo : 0;
  sp.g_hi = pf && epi == 3 ? a.g_hi : 0;
  for (int q = 0; q < 3; ++q) {
    sp.s_lo[q] = pf ? a.s_lo[q] : 0;
    sp.s_hi[q] = pf ? a.s_hi[q] : 0;
  }
  static const TmaMaps no_maps{};
  const TmaMaps& maps = a.maps ? *a.maps : no_maps;
  if (plan.vec) {
    switch (plan.chunks) {
      case 1: return launch_e<1, true>(epi, sp, maps, plan, s);
      case 2: return launch_e<2, true>(epi, sp, maps, plan, s);
      default: return launch_e<4, true>(epi, sp, maps, plan, s);
    }
  }
  switch (plan.chunks) {
    case 1: return launch_e<1, false>(epi, sp, maps, plan, s);
    case 2: return launch_e<2, false>(epi, sp, maps, plan, s);
    default: return launch_e<4, false>(epi, sp, maps, plan, s);
  }
}

}  // namespace bspmm
