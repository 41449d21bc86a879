// gcn_fused.cu — the fused batched graph-convolution layer (SURVEY §8(f)
// NEXT-1) on the 5th-generation tensor cores:
//
//     Y = sum_ch A_ch (X W_ch + 1 b_ch^T)        (PAPER.md Fig.
//     algo:graph_conv_batched, :304-321; Eq. (2), :66-68)
//
// The paper runs MatMul, Add and a Batched SpMM per channel plus an
// ElementWiseAdd (3 x channels + 1 launches, with U = X W_ch through HBM).
// Here the layer is ONE tensor-core GEMM per output tile, by associativity
// and distributivity (exact identities, R26):
//
//     Y = [A_1 X | ... | A_C X | r_1 ... r_C] . [W_1; ...; W_C; b_1^T; ...; b_C^T]
//
// with r_ch = rowsum(A_ch) (A_ch (1 b^T) = r_ch b^T).  The virtual left
// operand Z = [A_ch X | r] never exists in memory: per 32-column K block the
// math warps compute it from the X rows of the tile's graphs (staged by TMA
// in shared memory) with the SWA row loop of the Batched SpMM (fp32 FMA in
// CSR storage order) and write it straight into the
// swizzled operand layout the tensor core reads; the channel sum and the bias
// are part of the MMA's K reduction, accumulated in TMEM.  One launch per
// layer plus a small preparation launch (W transposed to K-major + split, and
// the tile -> first-graph table).
//
// Precision (bspmm_set_gcn_math): BSPMM_GCN_FP32 (default) = 3xTF32: each of
// Z and W split into hi = TF32-truncated and lo = the fp32 remainder, three
// MMAs (hi.hi + hi.lo + lo.hi) per K step -- ~2^-21 relative per product,
// fp32-accurate; BSPMM_GCN_TF32 = one MMA on the fp32 values (TF32 inputs);
// BSPMM_GCN_BF16 = one MMA on operands rounded to BF16 (exactly representable
// in TF32, so the products are those of a BF16 MMA; it runs at the TF32 rate).
//
// CTA (192 threads) per output tile = 128 node rows x nt output features:
//   warp 0      TMA producer: X halo blocks (rows of the graphs touching the
//               tile, 32 columns) and W blocks (hi / lo), mbarrier rings;
//   warp 1      TMEM allocation and the single-thread tcgen05.mma issuer;
//   warps 2-5   Z producers (SpMM into the swizzled operand), then the
//               epilogue (tcgen05.ld -> registers -> global stores).
#include <algorithm>
#include <cstdint>

#include <cuda_bf16.h>

#include "internal.h"
#include "ptx.cuh"

namespace bspmm {

constexpr int kGM = 128;          // node rows per tile (MMA M, TMEM lanes)
constexpr int kGK = 32;           // K per block: 32 x 4 B = one 128-byte swizzle row
constexpr int kGMath = 4;         // math warps per group (one per TMEM lane quarter)
// CTA size with NG groups of Z-producer warps (the groups take K blocks kb % NG)
__host__ __device__ constexpr int gcn_threads(int NG) { return 64 + 32 * kGMath * NG; }
constexpr int kXBox = 64;         // rows per X TMA box
constexpr int kZCol = 256;        // first TMEM column of the Z stages (after the accumulator, nt <= 256)

struct GcnParams {
  int32_t batch, channels, n_x, k;
  int32_t KX, nxb, nbias, ktot;   // K layout: channel ch's X block xb at ch*KX + 32 xb; bias blocks after C*KX
  int32_t nt, ntiles_n, tiles_m;  // output features per tile, feature tiles, row tiles
  int64_t N;                      // total rows
  int32_t mode;                   // 0 3xTF32, 1 TF32, 2 BF16-rounded
  int32_t xr, cap_e;              // staged X halo rows, staged structure entries (all channels)
  int32_t ws, zs, xs;             // ring depths (W, Z, X)
  int32_t w_stage, z_stage, x_stage;  // bytes per stage
  int32_t off_w, off_z, off_x, off_rp, off_col, off_val, off_rb, off_bar;
  uint32_t idesc;
  int32_t dbg;                    // 1 = no Z arithmetic, 2 = no MMAs (timing only, results undefined); 4 = 2 groups
  const int64_t* __restrict__ row_off;
  const int32_t* __restrict__ sizes;
  const int32_t* __restrict__ row_ptr;  // [channels][N + 1]
  const int32_t* __restrict__ col;
  const float* __restrict__ vals;
  const float* __restrict__ X;
  int64_t ldx;
  float* __restrict__ Y;
  int64_t ldy;
  const int32_t* __restrict__ gfirst;   // [tiles_m]: graph owning row 128 t
};

struct GcnMaps {
  CUtensorMap x;    // X [N x n_x], box {32, 64}, 128-byte swizzle (16-byte chunk j of row x at j ^ (x % 8))
  CUtensorMap whi;  // Wt_hi [k x ktot] (K-major), box {32, nt}, 128-byte swizzle
  CUtensorMap wlo;  // Wt_lo
};

__device__ __forceinline__ float tf32_hi(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

// CG = 2: a CTA pair (cluster of two) per 256-row tile -- each CTA forms the
// Z operand of its 128 rows in its own TMEM and stages HALF of the W block
// (nt / 2 output features) in its shared memory; the leader's single thread
// issues tcgen05.mma.cta_group::2 (M = 256), which reads both CTAs' Z and both
// W halves, so each SM's tensor core reads half the W bytes per K step from
// its shared memory.  Both CTAs' W loads complete on the leader's barrier; the
// peer's Z producers arrive on the leader's Z barrier; the leader's commits
// arrive on both CTAs' barriers.
template <int NG, int CG>
__global__ void __launch_bounds__(gcn_threads(NG), 1) gcn_fused_kernel(const GcnParams p,
                                                                     const __grid_constant__ GcnMaps m) {
  constexpr int kGGroups = NG;
  constexpr int kGThreads = gcn_threads(NG);
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte aligned base (128-byte swizzle atoms), by an offset on the shared
  // pointer itself so that every access below compiles to LDS/STS (an integer
  // round trip would make them generic loads and stores)
  unsigned char* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  __shared__ uint32_t s_tmem;
  __shared__ int64_t s_xlo;
  __shared__ int32_t s_xrows, s_staged_x, s_staged_s;
  __shared__ int32_t s_ebase[33];       // per channel: first staged entry (channels <= 32 staged)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  const uint32_t pair = CG == 2 ? blockIdx.x >> 1 : blockIdx.x;
  const int32_t tmp = (int32_t)(pair / (uint32_t)p.ntiles_n);
  const int32_t tn = (int32_t)(pair - (uint32_t)tmp * (uint32_t)p.ntiles_n);
  const int32_t tm = CG == 2 ? 2 * tmp + (int32_t)rank : tmp;
  const bool has_rows = tm < p.tiles_m;  // CG = 2, odd tile count: the last pair's second CTA has none
  const int64_t r0 = (int64_t)tm * kGM;
  const int32_t n0 = tn * p.nt;
  uint64_t* w_full = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* w_empty = w_full + p.ws;
  uint64_t* z_full = w_empty + p.ws;
  uint64_t* z_empty = z_full + p.zs;
  uint64_t* x_full = z_empty + p.zs;
  uint64_t* x_empty = x_full + p.xs;
  uint64_t* acc_full = x_empty + p.xs;
  int32_t* rbase = reinterpret_cast<int32_t*>(smem + p.off_rb);   // [128] halo row of the row's graph base, -1 = none
  int32_t* rp_s = reinterpret_cast<int32_t*>(smem + p.off_rp);    // [channels][129] staged entry index
  int32_t* col_s = reinterpret_cast<int32_t*>(smem + p.off_col);
  float* val_s = reinterpret_cast<float*>(smem + p.off_val);
  // TMEM: accumulator columns [0, nt), Z stages from column kZCol (hi, then lo
  // in 3xTF32), 32 columns of fp32 each; the whole 512 columns (1 CTA per SM)
  const uint32_t tmem_cols = 512u;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.ws; ++s) mbar_init(&w_full[s], 1), mbar_init(&w_empty[s], 1);
    for (int s = 0; s < p.zs; ++s) mbar_init(&z_full[s], kGMath * CG), mbar_init(&z_empty[s], 1);
    for (int s = 0; s < p.xs; ++s) mbar_init(&x_full[s], 1), mbar_init(&x_empty[s], kGGroups * kGMath);
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane < 3) prefetch_tensormap(lane == 0 ? (const void*)&m.x : lane == 1 ? (const void*)&m.whi : (const void*)&m.wlo);
  if (warp == 1) {
    if (CG == 2) tmem_alloc2(&s_tmem, tmem_cols);
    else tmem_alloc(&s_tmem, tmem_cols);
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync_all();  // the peer's barriers exist before any remote arrive / copy
  tc_fence_after();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // ---- tile setup: the graphs covering rows [r0, r0 + 128), the X halo, the structure
  const int32_t rows_in = !has_rows ? 0 : (int32_t)(p.N - r0 < kGM ? p.N - r0 : kGM);
  for (int r = threadIdx.x; r < kGM; r += kGThreads) rbase[r] = -1;
  __syncthreads();
  if (warp == 2 && !has_rows) {
    if (lane == 0) {
      s_xlo = 0;
      s_xrows = 0;
      s_staged_x = 1;
    }
  } else if (warp == 2) {
    const int32_t g0 = p.gfirst[tm];
    const int64_t xlo = p.row_off[g0];
    int64_t xhi = xlo;
    for (int32_t gb = g0;; gb += 32) {
      const int32_t g = gb + lane;
      int64_t ro = INT64_MAX;
      int32_t n = 0;
      if (g < p.batch) {
        ro = p.row_off[g];
        n = p.sizes ? p.sizes[g] : (int32_t)(p.row_off[g + 1] - ro);
      }
      const bool in = ro < r0 + kGM;
      if (in && n > 0) {
        xhi = max(xhi, ro + n);
        const int64_t a = max(ro, r0), b = min(ro + n, r0 + kGM);
        for (int64_t r = a; r < b; ++r) rbase[r - r0] = (int32_t)(ro - xlo);
      }
      if (__ballot_sync(0xffffffffu, in && g < p.batch) != 0xffffffffu) break;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) xhi = max(xhi, __shfl_xor_sync(0xffffffffu, xhi, d));
    if (lane == 0) {
      s_xlo = xlo;
      s_xrows = (int32_t)(xhi - xlo);
      s_staged_x = (xhi - xlo) <= p.xr ? 1 : 0;
    }
  } else if (warp == 3) {
    // per-channel entry ranges of the tile's rows; stage when they fit
    int32_t tot = 0;
    for (int32_t c0 = 0; c0 < p.channels; c0 += 32) {
      const int32_t ch = c0 + lane;
      int32_t cnt = 0;
      if (ch < p.channels && has_rows) {
        const int32_t* rp = p.row_ptr + (int64_t)ch * (p.N + 1) + r0;
        cnt = rp[rows_in] - rp[0];
      }
      int32_t incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int32_t v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
      }
      if (ch < p.channels && ch < 32) s_ebase[ch] = tot + incl - cnt;
      tot += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
      s_staged_s = (p.channels <= 32 && tot <= p.cap_e) ? 1 : 0;
      if (p.channels <= 32) s_ebase[min(p.channels, 32)] = tot;
    }
  }
  __syncthreads();
  const bool staged_s = s_staged_s != 0;
  if (staged_s && warp >= 2 && has_rows) {  // the math warps stage row pointers, columns and values
    const int mt = threadIdx.x - 64, MT = kGThreads - 64;
    for (int32_t ch = 0; ch < p.channels; ++ch) {
      const int32_t* rp = p.row_ptr + (int64_t)ch * (p.N + 1) + r0;
      const int32_t e0 = rp[0];
      const int32_t eb = s_ebase[ch];
      for (int r = mt; r <= kGM; r += MT) rp_s[ch * (kGM + 1) + r] = eb + (r <= rows_in ? rp[r] - e0 : rp[rows_in] - e0);
      const int32_t ne = s_ebase[ch + 1] - eb;
      for (int32_t e = mt; e < ne; e += MT) {
        col_s[eb + e] = p.col[e0 + e];
        val_s[eb + e] = p.vals[e0 + e];
      }
    }
  }
  __syncthreads();
  if (staged_s && warp >= 2 && warp < 2 + kGMath) {  // entries of row r: col -> halo row (rbase[r] + col)
    const int r = threadIdx.x - 64;
    const int32_t rb = rbase[r];
    if (rb >= 0)
      for (int32_t ch = 0; ch < p.channels; ++ch)
        for (int32_t e = rp_s[ch * (kGM + 1) + r]; e < rp_s[ch * (kGM + 1) + r + 1]; ++e) col_s[e] += rb;
  }
  __syncthreads();
  const int64_t xlo = s_xlo;
  const bool staged_x = s_staged_x != 0;
  const int32_t nkb = p.nxb * p.channels + p.nbias;

  if (warp == 0) {
    // ======== TMA producer ========
    if (lane == 0) {
      int wsi = 0, xsi = 0;
      uint32_t wph = 0, xph = 0;
      // CG = 2: this CTA's half of the W block (nt / 2 features), its bytes
      // completing on the leader's barrier, which the leader arms for both halves
      const uint32_t wbytes = (uint32_t)p.nt * 128u * (p.mode == 0 ? 2u : 1u);
      const int32_t nh = p.nt / CG;
      const int32_t nbox = (s_xrows + kXBox - 1) / kXBox;
      auto issue_w = [&](int32_t kcoord) {
        mbar_wait(&w_empty[wsi], wph ^ 1u);
        unsigned char* st = smem + p.off_w + (size_t)wsi * p.w_stage;
        if (CG == 2) {
          const uint32_t lb = mapa_rank(&w_full[wsi], 0);
          if (rank == 0) mbar_arrive_expect_tx(&w_full[wsi], wbytes);
          const int32_t y = n0 + (int32_t)rank * nh;
          tma2_load_2d(st, &m.whi, kcoord, y, lb);
          if (p.mode == 0) tma2_load_2d(st + (size_t)nh * 128, &m.wlo, kcoord, y, lb);
        } else {
          mbar_arrive_expect_tx(&w_full[wsi], wbytes);
          tma_load_2d(st, &m.whi, kcoord, n0, &w_full[wsi]);
          if (p.mode == 0) tma_load_2d(st + (size_t)p.nt * 128, &m.wlo, kcoord, n0, &w_full[wsi]);
        }
        if (++wsi == p.ws) wsi = 0, wph ^= 1u;
      };
      for (int32_t xb = 0; xb < p.nxb; ++xb) {
        mbar_wait(&x_empty[xsi], xph ^ 1u);
        if (staged_x && nbox > 0) {
          unsigned char* xs = smem + p.off_x + (size_t)xsi * p.x_stage;
          mbar_arrive_expect_tx(&x_full[xsi], (uint32_t)nbox * kXBox * 128u);
          for (int32_t j = 0; j < nbox; ++j)
            tma_load_2d(xs + (size_t)j * kXBox * 128, &m.x, xb * kGK, (int32_t)(xlo + (int64_t)j * kXBox), &x_full[xsi]);
        } else {
          mbar_arrive(&x_full[xsi]);
        }
        if (++xsi == p.xs) xsi = 0, xph ^= 1u;
        for (int32_t ch = 0; ch < p.channels; ++ch) issue_w(ch * p.KX + xb * kGK);
      }
      for (int32_t j = 0; j < p.nbias; ++j) issue_w(p.channels * p.KX + j * kGK);
    }
  } else if (warp == 1) {
    // ======== MMA issuer (one thread; CG = 2: the leader CTA's) ========
    if (lane == 0 && (CG == 1 || rank == 0)) {
      const uint32_t d = s_tmem;
      int wsi = 0, zsi = 0;
      uint32_t wph = 0, zph = 0;
      for (int32_t kb = 0; kb < nkb; ++kb) {
        mbar_wait(&w_full[wsi], wph);
        mbar_wait(&z_full[zsi], zph);
        tc_fence_after();
        unsigned char* ws = smem + p.off_w + (size_t)wsi * p.w_stage;
        const uint64_t wh = smem_desc_sw128(ws), wl = smem_desc_sw128(ws + (size_t)(p.nt / CG) * 128);
        const uint32_t zh = d + kZCol + (uint32_t)zsi * (p.mode == 0 ? 64u : 32u), zl = zh + 32u;
#pragma unroll
        for (int j = 0; j < kGK / 8 && !(p.dbg & 2); ++j) {  // UMMA_K = 8: 8 TMEM columns of A, +32 bytes of B
          if (CG == 2) {
            mma2_tf32_ts(d, zh + 8 * j, wh + 2 * j, p.idesc, (kb | j) != 0);
            if (p.mode == 0) {
              mma2_tf32_ts(d, zh + 8 * j, wl + 2 * j, p.idesc, 1u);
              mma2_tf32_ts(d, zl + 8 * j, wh + 2 * j, p.idesc, 1u);
            }
          } else {
            mma_tf32_ts(d, zh + 8 * j, wh + 2 * j, p.idesc, (kb | j) != 0);
            if (p.mode == 0) {
              mma_tf32_ts(d, zh + 8 * j, wl + 2 * j, p.idesc, 1u);
              mma_tf32_ts(d, zl + 8 * j, wh + 2 * j, p.idesc, 1u);
            }
          }
        }
        if (CG == 2) {
          mma2_commit_both(&w_empty[wsi]);
          mma2_commit_both(&z_empty[zsi]);
        } else {
          mma_commit(&w_empty[wsi]);
          mma_commit(&z_empty[zsi]);
        }
        if (++wsi == p.ws) wsi = 0, wph ^= 1u;
        if (++zsi == p.zs) zsi = 0, zph ^= 1u;
      }
      if (CG == 2) mma2_commit_both(acc_full);
      else mma_commit(acc_full);
    }
  } else {
    // ======== math warps: Z = [A_ch X | rowsums] block by block ========
    // lane = row: each lane forms its own row's 32 K columns in registers
    // (the SWA row loop over its entries, fp32 FMA in storage order, PAPER.md
    // :196-207), reading whole 128-byte X rows (swizzled like the operand
    // tiles) and writing one 128-byte swizzled row of Z -- no cross-lane
    // dependence, all loads of an entry in flight at once
    const int q = warp & 3;      // the TMEM lane quarter this warp may access
    const int r = q * 32 + lane;  // its row (= TMEM lane) of the tile
    const int32_t rb = rbase[r];
    const uint32_t tq = s_tmem + ((uint32_t)(q * 32) << 16);
    // NG groups of four warps take K blocks in turn (kb % NG): while one group
    // forms Z block kb, the others form kb + 1, ...
    const int grp = (warp - 2) / kGMath;
    auto row_range = [&](int32_t ch, int32_t& e0, int32_t& e1) {
      if (staged_s) {
        e0 = rp_s[ch * (kGM + 1) + r];
        e1 = rp_s[ch * (kGM + 1) + r + 1];
      } else {
        const int32_t* rp = p.row_ptr + (int64_t)ch * (p.N + 1) + r0 + r;
        e0 = rp[0];
        e1 = rp[1];
      }
    };
    // Z row -> TMEM stage zsi (hi = TF32 truncation, lo = the fp32 remainder in
    // 3xTF32; BF16 mode: rounded to BF16), then make it visible to the MMA
    // the Z stage is ready: arrive on the MMA issuer's barrier (CG = 2: the leader's)
    auto z_arrive = [&](int zsi_) {
      if (CG == 2) mbar_arrive_cluster(mapa_rank(&z_full[zsi_], 0));
      else mbar_arrive(&z_full[zsi_]);
    };
    auto put_row = [&](int zsi_, float (&z)[32]) {
      const uint32_t col = kZCol + (uint32_t)zsi_ * (p.mode == 0 ? 64u : 32u);
      if (p.mode == 0) {
        float lo[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float h = tf32_hi(z[c]);
          lo[c] = z[c] - h;
          z[c] = h;
        }
        tmem_st32(tq + col + 32u, lo);
      } else if (p.mode == 2) {
#pragma unroll
        for (int c = 0; c < 32; ++c) z[c] = __bfloat162float(__float2bfloat16_rn(z[c]));
      }
      tmem_st32(tq + col, z);
      tmem_wait_st();
      tc_fence_before();
    };
    for (int32_t xb = 0; xb < p.nxb; ++xb) {
      const int xsi = xb % p.xs;
      const unsigned char* xs = smem + p.off_x + (size_t)xsi * p.x_stage;
      bool waited_x = false;
      for (int32_t ch = 0; ch < p.channels; ++ch) {
        const int32_t kb = xb * p.channels + ch;
        if (kb % kGGroups != grp) continue;
        const int zsi = kb % p.zs;
        if (!waited_x) {
          mbar_wait(&x_full[xsi], (uint32_t)(xb / p.xs) & 1u);
          waited_x = true;
        }
        mbar_wait(&z_empty[zsi], ((uint32_t)(kb / p.zs) & 1u) ^ 1u);
        tc_fence_after();
        float z[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) z[c] = 0.f;
        if (rb >= 0 && !(p.dbg & 1)) {
          int32_t e, e1;
          row_range(ch, e, e1);
          if (staged_s && staged_x) {
            // two entries per iteration: both X rows' loads in flight before
            // the FMAs, which stay in storage order (entry e, then e + 1)
            auto xrow4 = [&](int32_t xr, int j) {
              return *reinterpret_cast<const float4*>(xs + (size_t)xr * 128 + ((j ^ (xr & 7)) << 4));
            };
            for (; e + 1 < e1; e += 2) {
              const int32_t xr0 = col_s[e], xr1 = col_s[e + 1];  // halo rows (staged)
              const float a0 = val_s[e], a1 = val_s[e + 1];
              float4 v0[8], v1[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) v0[j] = xrow4(xr0, j), v1[j] = xrow4(xr1, j);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                z[4 * j] = fmaf(a0, v0[j].x, z[4 * j]);
                z[4 * j + 1] = fmaf(a0, v0[j].y, z[4 * j + 1]);
                z[4 * j + 2] = fmaf(a0, v0[j].z, z[4 * j + 2]);
                z[4 * j + 3] = fmaf(a0, v0[j].w, z[4 * j + 3]);
                z[4 * j] = fmaf(a1, v1[j].x, z[4 * j]);
                z[4 * j + 1] = fmaf(a1, v1[j].y, z[4 * j + 1]);
                z[4 * j + 2] = fmaf(a1, v1[j].z, z[4 * j + 2]);
                z[4 * j + 3] = fmaf(a1, v1[j].w, z[4 * j + 3]);
              }
            }
            if (e < e1) {
              const int32_t xr0 = col_s[e];
              const float a0 = val_s[e];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 v = xrow4(xr0, j);
                z[4 * j] = fmaf(a0, v.x, z[4 * j]);
                z[4 * j + 1] = fmaf(a0, v.y, z[4 * j + 1]);
                z[4 * j + 2] = fmaf(a0, v.z, z[4 * j + 2]);
                z[4 * j + 3] = fmaf(a0, v.w, z[4 * j + 3]);
              }
            }
          } else {
            for (; e < e1; ++e) {
              const int32_t xr = staged_s ? col_s[e] : rb + p.col[e];  // staged: halo row already
              const float a = staged_s ? val_s[e] : p.vals[e];
              if (staged_x) {
                const unsigned char* xrow = xs + (size_t)xr * 128;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  const float4 v = *reinterpret_cast<const float4*>(xrow + ((j ^ (xr & 7)) << 4));
                  z[4 * j] = fmaf(a, v.x, z[4 * j]);
                  z[4 * j + 1] = fmaf(a, v.y, z[4 * j + 1]);
                  z[4 * j + 2] = fmaf(a, v.z, z[4 * j + 2]);
                  z[4 * j + 3] = fmaf(a, v.w, z[4 * j + 3]);
                }
              } else {
                const float* xg = p.X + (xlo + xr) * p.ldx + xb * kGK;
#pragma unroll
                for (int c = 0; c < 32; ++c) z[c] = fmaf(a, xb * kGK + c < p.n_x ? __ldg(xg + c) : 0.f, z[c]);
              }
            }
          }
        }
        put_row(zsi, z);
        __syncwarp();
        if (lane == 0) z_arrive(zsi);
      }
      // both groups release every X block (a group with no K block in it too;
      // the X ring then never runs ahead of either)
      if (!waited_x) mbar_wait(&x_full[xsi], (uint32_t)(xb / p.xs) & 1u);
      __syncwarp();
      if (lane == 0) mbar_arrive(&x_empty[xsi]);
    }
    for (int32_t j = 0; j < p.nbias; ++j) {  // K columns C*KX + 32 j + c: rowsum of channel 32 j + c
      const int32_t kb = p.nxb * p.channels + j;
      if (kb % kGGroups != grp) continue;
      const int zsi = kb % p.zs;
      mbar_wait(&z_empty[zsi], ((uint32_t)(kb / p.zs) & 1u) ^ 1u);
      tc_fence_after();
      float z[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        float sum = 0.f;
        const int32_t ch = j * 32 + c;
        if (rb >= 0 && ch < p.channels) {
          int32_t e, e1;
          row_range(ch, e, e1);
          for (; e < e1; ++e) sum += staged_s ? val_s[e] : p.vals[e];
        }
        z[c] = sum;
      }
      put_row(zsi, z);
      __syncwarp();
      if (lane == 0) z_arrive(zsi);
    }
    // ======== epilogue: TMEM -> registers -> Y ========
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const int re = q * 32 + lane;
    const int64_t g = r0 + re;
    const bool live = re < rows_in && rbase[re] >= 0;
    const bool vec = ((p.ldy & 3) == 0) && ((reinterpret_cast<uintptr_t>(p.Y) & 15) == 0);
    float* yrow = p.Y + g * p.ldy;
    const int32_t part = ((p.nt + kGGroups - 1) / kGGroups + 15) & ~15;  // group g: columns [g part, (g+1) part)
    for (int32_t c0 = grp * part; c0 < min(p.nt, (grp + 1) * part); c0 += 16) {
      float v[16];
      tmem_ld16(s_tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);  // whole warp, converged
      const int32_t cg = n0 + c0;
      if (live && cg < p.k) {
        if (vec && cg + 16 <= p.k) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            stg_cs_f4(yrow + cg + 4 * u, make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]));
        } else {
#pragma unroll
          for (int u = 0; u < 16; ++u)
            if (cg + u < p.k) yrow[cg + u] = v[u];
        }
      }
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) {
    cluster_sync_all();  // neither CTA frees its TMEM while the pair's MMAs may read it
    if (warp == 1) tmem_dealloc2(s_tmem, tmem_cols);
  } else if (warp == 1) {
    tmem_dealloc(s_tmem, tmem_cols);
  }
}

// ---- preparation: W -> K-major (transposed, padded, split), bias rows, and
// the tile -> first-graph table
struct GcnPrep {
  int32_t batch, channels, n_x, k, KX, ktot, mode, tiles_m;
  int64_t N;
  int32_t wblocks_c, wblocks_k;  // transpose tiles: ceil(k / 32) x (ktot / 32)
  const float* W;
  const float* bias;
  float* whi;
  float* wlo;
  const int64_t* row_off;
  int32_t* gfirst;
};

__device__ __forceinline__ void split_store(const GcnPrep& q, int64_t idx, float v) {
  if (q.mode == 0) {
    const float h = tf32_hi(v);
    q.whi[idx] = h;
    q.wlo[idx] = v - h;
  } else if (q.mode == 1) {
    q.whi[idx] = v;
  } else {
    q.whi[idx] = __bfloat162float(__float2bfloat16_rn(v));
  }
}

__global__ void __launch_bounds__(256) gcn_prep_kernel(const GcnPrep q) {
  __shared__ float tile[32][33];
  const int32_t nwb = q.wblocks_c * q.wblocks_k;
  if ((int32_t)blockIdx.x < nwb) {
    // output tile: Wt rows c0 .. c0+32 (features), K columns kk0 .. kk0+32
    const int32_t bc = blockIdx.x % q.wblocks_c, bk = blockIdx.x / q.wblocks_c;
    const int32_t c0 = bc * 32, kk0 = bk * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 32
    const int32_t cx = q.channels * q.KX;
    for (int i = ty; i < 32; i += 8) {  // read along the feature index c (coalesced in W)
      const int32_t kk = kk0 + i, c = c0 + tx;
      float v = 0.f;
      if (c < q.k) {
        if (kk < cx) {
          const int32_t ch = kk / q.KX, l = kk - ch * q.KX;
          if (l < q.n_x) v = q.W[((int64_t)ch * q.n_x + l) * q.k + c];
        } else if (q.bias && kk - cx < q.channels) {
          v = q.bias[(int64_t)(kk - cx) * q.k + c];
        }
      }
      tile[i][tx] = v;
    }
    __syncthreads();
    for (int j = ty; j < 32; j += 8) {  // write along K (coalesced in Wt)
      const int32_t c = c0 + j;
      if (c < q.k) split_store(q, (int64_t)c * q.ktot + kk0 + tx, tile[tx][j]);
    }
    return;
  }
  // tile table: graph i covers rows [row_off[i], row_off[i+1]) (graph 0 also
  // the rows before it, the last graph the rows up to N); gfirst[t] = the
  // graph covering row 128 t
  const int64_t i = (int64_t)(blockIdx.x - nwb) * blockDim.x + threadIdx.x;
  if (i >= q.batch) return;
  const int64_t lo = i == 0 ? 0 : q.row_off[i];
  const int64_t hi = i == q.batch - 1 ? max(q.N, q.row_off[i + 1]) : q.row_off[i + 1];
  for (int64_t t = (lo + kGM - 1) / kGM; t * kGM < hi && t < q.tiles_m; ++t) q.gfirst[t] = (int32_t)i;
}

// X with a leading dimension TMA cannot address (ldx % 4 != 0, or misaligned):
// a packed copy with ld = n_x rounded up to 4
__global__ void __launch_bounds__(256) gcn_pack_x_kernel(const float* __restrict__ X, int64_t ldx, int32_t n_x,
                                                         int64_t N, float* __restrict__ out, int64_t ldo) {
  const int64_t total = N * ldo;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / ldo, c = idx - r * ldo;
    out[idx] = c < n_x ? X[r * ldx + c] : 0.f;
  }
}

bool plan_gcn(int32_t channels, int32_t n_x, int32_t k, int64_t N, int32_t max_rows, int32_t smem_optin, int32_t mode,
              int32_t num_sms, int32_t nt_override, int32_t cg, GcnPlan* out) {
  GcnPlan L{};
  L.cg = cg == 2 ? 2 : 1;
  L.KX = (n_x + kGK - 1) / kGK * kGK;
  L.nxb = L.KX / kGK;
  L.nbias = (channels + 31) / 32;
  L.ktot = channels * L.KX + L.nbias * kGK;
  // output features per tile (MMA N, TMEM accumulator columns): up to 256, so
  // that k = 512 takes two feature tiles (Z is formed once per feature tile);
  // 128 when 256-wide tiles would leave SMs idle (small batches: more CTAs,
  // each forming its Z again; Reaction100-like 86 -> 70 us, 64-wide tiles
  // measured slower again, 131 us)
  L.tiles_m = (int32_t)((N + kGM - 1) / kGM);
  L.nt = k > 128 ? 256 : (k > 64 ? 128 : (k > 32 ? 64 : 32));
  if (L.nt == 256 && (int64_t)L.tiles_m * ((k + 255) / 256) < num_sms) L.nt = 128;
  if (nt_override >= 32 && nt_override <= 256) L.nt = nt_override;
  if (L.cg == 2 && L.nt < 64) L.cg = 1;  // a CTA pair splits the features: nt / 2 >= 32 (one 128-byte row group)
  L.ntiles_n = (k + L.nt - 1) / L.nt;
  const int64_t R = max_rows > 0 ? max_rows : 64;
  L.xr = (int32_t)std::min<int64_t>(256, (kGM + 2 * (R - 1) + kXBox - 1) / kXBox * kXBox);
  const int32_t split = mode == 0 ? 2 : 1;
  L.w_stage = L.nt / L.cg * 128 * split;  // CG = 2: this CTA's half of the features
  L.z_stage = 0;  // Z lives in TMEM (32 columns per stage and split part)
  L.x_stage = L.xr * 128;
  L.ws = 4;
  L.zs = std::min(8, (512 - kZCol) / (32 * split));
  L.xs = 2;
  auto layout = [&]() {
    int32_t off = 0;
    L.off_w = off;
    off += L.ws * L.w_stage;
    L.off_z = off;
    off += L.zs * L.z_stage;
    L.off_x = off;
    off += L.xs * L.x_stage;
    L.off_rb = off;
    off += kGM * 4;
    L.off_bar = off;
    off += 8 * (2 * L.ws + 2 * L.zs + 2 * L.xs + 1);
    off = (off + 15) / 16 * 16;
    L.off_rp = off;
    off += std::min(channels, 32) * (kGM + 1) * 4;
    off = (off + 15) / 16 * 16;
    const int32_t room = smem_optin - 2048 - off;  // 1024 alignment slack of the dynamic base, 1024 static + reserve
    L.cap_e = std::max(0, std::min(8192, room / 8));
    L.off_col = off;
    off += L.cap_e * 4;
    L.off_val = off;
    off += L.cap_e * 4;
    L.smem = off + 1024;
  };
  layout();
  while (L.cap_e < 2048 && L.ws > 2) {  // room for the structure first
    --L.ws;
    layout();
  }
  if (L.cap_e < 256 && L.xs > 1) {
    L.xs = 1;
    layout();
  }
  if (L.smem > smem_optin) return false;
  // instruction descriptor: D fp32, A = B = TF32, both K-major, M = 128 (256
  // for a CTA pair), N = nt
  L.idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(L.nt >> 3) << 17) |
            ((uint32_t)((kGM * L.cg) >> 4) << 24);
  *out = L;
  return true;
}

cudaError_t launch_gcn_prep(const GcnPlan& L, int32_t batch, int32_t channels, int32_t n_x, int32_t k, int64_t N,
                            int32_t mode, const float* W, const float* bias, float* whi, float* wlo,
                            const int64_t* row_off, int32_t* gfirst, cudaStream_t s) {
  GcnPrep q;
  q.batch = batch;
  q.channels = channels;
  q.n_x = n_x;
  q.k = k;
  q.KX = L.KX;
  q.ktot = L.ktot;
  q.mode = mode;
  q.tiles_m = L.tiles_m;
  q.N = N;
  q.wblocks_c = (k + 31) / 32;
  q.wblocks_k = L.ktot / 32;
  q.W = W;
  q.bias = bias;
  q.whi = whi;
  q.wlo = wlo;
  q.row_off = row_off;
  q.gfirst = gfirst;
  const int64_t blocks = (int64_t)q.wblocks_c * q.wblocks_k + (batch + 255) / 256;
  gcn_prep_kernel<<<(unsigned)blocks, 256, 0, s>>>(q);
  return cudaGetLastError();
}

cudaError_t launch_gcn_pack_x(const float* X, int64_t ldx, int32_t n_x, int64_t N, float* out, int64_t ldo,
                              int32_t num_sms, cudaStream_t s) {
  gcn_pack_x_kernel<<<num_sms * 8, 256, 0, s>>>(X, ldx, n_x, N, out, ldo);
  return cudaGetLastError();
}

cudaError_t launch_gcn_fused(const GcnPlan& L, const GcnArgs& a, cudaStream_t s) {
  GcnParams p;
  p.batch = a.batch;
  p.channels = a.channels;
  p.n_x = a.n_x;
  p.k = a.k;
  p.KX = L.KX;
  p.nxb = L.nxb;
  p.nbias = L.nbias;
  p.ktot = L.ktot;
  p.nt = L.nt;
  p.ntiles_n = L.ntiles_n;
  p.tiles_m = L.tiles_m;
  p.N = a.N;
  p.mode = a.mode;
  p.xr = L.xr;
  p.cap_e = L.cap_e;
  p.ws = L.ws;
  p.zs = L.zs;
  p.xs = L.xs;
  p.w_stage = L.w_stage;
  p.z_stage = L.z_stage;
  p.x_stage = L.x_stage;
  p.off_w = L.off_w;
  p.off_z = L.off_z;
  p.off_x = L.off_x;
  p.off_rp = L.off_rp;
  p.off_col = L.off_col;
  p.off_val = L.off_val;
  p.off_rb = L.off_rb;
  p.off_bar = L.off_bar;
  p.idesc = L.idesc;
  p.dbg = a.dbg;
  p.row_off = a.row_off;
  p.sizes = a.sizes;
  p.row_ptr = a.row_ptr;
  p.col = a.col;
  p.vals = a.vals;
  p.X = a.X;
  p.ldx = a.ldx;
  p.Y = a.Y;
  p.ldy = a.ldy;
  p.gfirst = a.gfirst;
  GcnMaps maps;
  maps.x = *a.map_x;
  maps.whi = *a.map_whi;
  maps.wlo = *a.map_wlo;
  // Z-producer groups: 3xTF32 2 (its tensor-core operand traffic bounds it;
  // a third group measured 6% slower), the one-pass modes 3; debug bit
  // 524288 swaps
  const int ng = ((a.mode == 0) != ((a.dbg & 4) != 0)) ? 2 : 3;
  const int cg = L.cg;
  auto kern = cg == 2 ? (ng == 2 ? gcn_fused_kernel<2, 2> : gcn_fused_kernel<3, 2>)
                      : (ng == 2 ? gcn_fused_kernel<2, 1> : gcn_fused_kernel<3, 1>);
  const int ki = (ng - 2) + 2 * (cg - 1);
  static thread_local int configured[4][64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured[ki][dev & 63] < L.smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.smem);
    if (e != cudaSuccess) return e;
    configured[ki][dev & 63] = L.smem;
  }
  // CG = 2: pairs of CTAs (tile rows 2t, 2t + 1) per feature tile
  const int64_t grid = cg == 2 ? 2 * ((int64_t)(L.tiles_m + 1) / 2) * L.ntiles_n : (int64_t)L.tiles_m * L.ntiles_n;
  if (grid == 0) return cudaSuccess;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(gcn_threads(ng));
  cfg.dynamicSmemBytes = L.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cg;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = cg == 2 ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, p, maps);
}

}  // namespace bspmm
