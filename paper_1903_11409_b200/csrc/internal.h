// internal.h — private declarations shared by the libbspmm.so sources.
#pragma once
#include <cuda.h>  // CUtensorMap type only; the encoder is fetched via cudaGetDriverEntryPoint
#include <cuda_runtime.h>

#include <string>

#include "bspmm.h"
#include "bspmm_debug.h"

#if defined(__CUDACC__)
#define BSPMM_HD __host__ __device__
#else
#define BSPMM_HD
#endif

namespace bspmm {

constexpr int kMaxStages = 8;
constexpr int kHdrBytes = 32;       // per-stage unit header
constexpr int kDefaultRows = 64;    // planning assumption when no max_rows hint
constexpr int kDefaultChunks = 2;   // column chunks per lane (fewer lanes per row, more rows per warp)
constexpr int kMaxVecKt = 512;      // 4 float4 chunks x 32 lanes
constexpr int kMaxScalarKt = 128;   // 4 float chunks x 32 lanes
constexpr int kCooSmemCap = 2048;   // default COO entries sorted in shared memory

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int32_t pow2_ceil(int32_t x) {
  int32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}
BSPMM_HD inline int32_t align_up(int32_t x, int32_t a) { return (x + a - 1) / a * a; }

// smem carve-up shared by planner and kernel: [hdr S*32][full S*8][empty S*8]
// [early 8][sfull S*8][cvt S*8] pad 128, then stages.  Per stage: header +
// "full" + "empty" barriers; one barrier for the first unit's early B tile
// (spmm_csr.cu early_b); fused COO mode, per stage: a "slice full" barrier
// (the raw SparseTensor slice lands on its own barrier) and a "converted"
// barrier (the converter warps have written the stage's CSR slice)
BSPMM_HD inline int32_t ring_prefix_bytes(int32_t stages) { return align_up(stages * (kHdrBytes + 32) + 8, 128); }
// fused COO mode: 20 warps per CTA (5 per SM sub-partition: 96 registers) --
// the producer, W consumer warps and 19 - W converter warps that convert the
// next unit's SparseTensor slice while the consumers compute the current one
// (spmm_csr.cu convert_units); W from the tuning knob, else kCooConsumers
constexpr int kCooWarps = 20;
constexpr int kCooConsumers = 10;
inline int32_t coo_consumer_warps(int32_t tune) { return tune > 0 ? (tune < 18 ? tune : 18) : kCooConsumers; }

// planner (plan.cpp)
bspmm_status_t make_plan(int32_t k, int32_t batch, bool aligned, int32_t max_rows, int64_t max_nnz,
                         int32_t num_sms, int32_t smem_per_cta, int32_t kt_override, int32_t warps,
                         int32_t ctas_per_sm, int32_t chunks_pref, bspmm_plan_t* out, bool coo = false);

// 2-D TMA descriptors over B [rows x k] (row pitch ldb) with box {kt, 2^b rows},
// b = 0..8: a unit of n_i rows is staged with popcount(n_i) tensor copies
constexpr int kTmaMaps = 9;
struct TmaMaps {
  CUtensorMap m[kTmaMaps];
};

struct CsrArgs {
  int32_t batch, k;
  const int64_t* row_off;
  const int32_t* sizes;
  const int32_t* row_ptr;
  const int32_t* col;
  const float* vals;
  const float* B;
  int64_t ldb;
  float* C;
  int64_t ldc;
  unsigned long long* trace;  // debug phase timestamps (bspmm_set_trace) or null
  int32_t dbg;                // debug bits (bspmm_set_debug)
  const TmaMaps* maps;        // non-null: full k-tiles are staged with 2-D tensor TMA
  const float* bias = nullptr;  // GCN epilogue: C += rowsum(A) (x) bias (k floats), or null
  int32_t accumulate = 0;       // GCN epilogue: C += previous C
  unsigned long long* sched = nullptr;  // dynamic-schedule ticket counter (device, zero between launches)
  const int64_t* coo_nnz_off = nullptr; // fused COO mode: per-matrix entry offsets (col/vals = raw COO)
  const int32_t* coo_idx = nullptr;     // fused COO mode: (row, col) pairs
  int* err = nullptr;                   // device error flag (bit 64: COO unit over stage capacity)
  int32_t cvt_warps = 0;                // fused COO mode: converter warps (coo_consumer_warps)
  int32_t mc = 0;                       // NEXT-4b: C is a multicast VA (multimem.st epilogue)
  const float* G = nullptr;             // SDDMM mode (NEXT-2): sd_out[e] = <G[row_e], B[col_e]>
  int64_t ldg = 0;
  float* sd_out = nullptr;
  // the allocation holding B ([b_lo, b_hi), 0 = unknown): pre-wait L2
  // prefetches of B are clipped to it
  uint64_t b_lo = 0, b_hi = 0;
  // the allocations of the structure arrays (CSR: row_ptr, col, vals; COO:
  // -, idx, vals), for the same prefetch of the matrix's structure
  uint64_t s_lo[3] = {}, s_hi[3] = {};
  uint64_t g_lo = 0, g_hi = 0;  // SDDMM mode: grad_C's allocation
};
// debug bit 16777216: no pre-wait L2 prefetch of B (tile kernels)
constexpr int32_t kDbgNoPrewaitPrefetch = 1 << 24;
// debug bit 33554432: the pre-wait prefetch covers B only (not the matrix's structure)
constexpr int32_t kDbgNoStructPrefetch = 1 << 25;
// debug bit 536870912: backward of streaming batches by the separate kernels
// (transpose + forward kernel, SDDMM) instead of the fused kernel
constexpr int32_t kDbgNoFusedBackward = 1 << 29;
// bspmm.cu: the device allocation containing p (queried per call); false if unknown
bool alloc_range(bspmm_handle_t h, const void* p, uint64_t* lo, uint64_t* hi);

// kernels (.cu)
cudaError_t launch_spmm_csr(const CsrArgs& a, const bspmm_plan_t& plan, cudaStream_t s);
// small-batch tile kernel (spmm_tile.cu): one CTA per (matrix, float4 column block)
struct TileLayout {
  int32_t cb, tiles, per_sm, smem;
  int32_t cap_rows, cap_nnz, rp_off, col_off, val_off;
  int32_t pair_off = 0, cval_off = 0, slot_off = 0, cnt_off = 0;  // SparseTensor conversion scratch
  int64_t units;
};
bool plan_tile(int32_t batch, int32_t k, int32_t max_rows, int64_t max_nnz, int32_t num_sms, int32_t cb_override,
               TileLayout* out, bool coo = false);
cudaError_t launch_spmm_tile(const CsrArgs& a, const TileLayout& L, cudaStream_t s);
// fused GCN layer on tcgen05 (gcn_fused.cu)
struct GcnPlan {
  int32_t KX, nxb, nbias, ktot, nt, ntiles_n, tiles_m, xr, cap_e;
  int32_t cg;  // 1: one CTA per 128-row tile; 2: a CTA pair per 256 rows (tcgen05 cta_group::2)
  int32_t ws, zs, xs, w_stage, z_stage, x_stage;
  int32_t off_w, off_z, off_x, off_rp, off_col, off_val, off_rb, off_bar, smem;
  uint32_t idesc;
};
struct GcnArgs {
  int32_t batch, channels, n_x, k, mode, dbg;
  int64_t N;
  const int64_t* row_off;
  const int32_t* sizes;
  const int32_t* row_ptr;
  const int32_t* col;
  const float* vals;
  const float* X;
  int64_t ldx;
  float* Y;
  int64_t ldy;
  const int32_t* gfirst;
  const CUtensorMap* map_x;
  const CUtensorMap* map_whi;
  const CUtensorMap* map_wlo;
};
bool plan_gcn(int32_t channels, int32_t n_x, int32_t k, int64_t N, int32_t max_rows, int32_t smem_optin, int32_t mode,
              int32_t num_sms, int32_t nt_override, int32_t cg, GcnPlan* out);
cudaError_t launch_gcn_prep(const GcnPlan& L, int32_t batch, int32_t channels, int32_t n_x, int32_t k, int64_t N,
                            int32_t mode, const float* W, const float* bias, float* whi, float* wlo,
                            const int64_t* row_off, int32_t* gfirst, cudaStream_t s);
cudaError_t launch_gcn_pack_x(const float* X, int64_t ldx, int32_t n_x, int64_t N, float* out, int64_t ldo,
                              int32_t num_sms, cudaStream_t s);
cudaError_t launch_gcn_fused(const GcnPlan& L, const GcnArgs& a, cudaStream_t s);
// decoupled look-back scan state (persistent per handle; epoch-tagged, never reset per call)
struct ScanState {
  uint32_t* flags;                 // [tiles] (epoch << 2) | {1: aggregate, 2: inclusive}
  int64_t* agg;                    // [tiles]
  int64_t* incl;                   // [tiles]
  unsigned long long* ticket;      // tile ticket counter (0 between launches: self-resetting)
  uint32_t epoch;                  // 1 .. 2^30-1
};
int32_t scan_tiles(int32_t batch);
cudaError_t launch_offsets(int32_t batch, const int32_t* sizes, int64_t* out, const ScanState& st,
                           cudaStream_t s);
cudaError_t launch_coo2csr(int32_t batch, const int64_t* row_off, const int32_t* sizes,
                           const int64_t* nnz_off, const int32_t* idx, const float* vals, int32_t* row_ptr,
                           int32_t* col_out, float* val_out, uint64_t* ws_keys, uint32_t* ws_pay,
                           int64_t ws_stride, int32_t smem_cap, cudaStream_t s);
int32_t coo_smem_cap(int64_t max_nnz_hint, int32_t smem_optin);
cudaError_t launch_spmm_coo_atomic(int32_t batch, int32_t k, const int64_t* row_off, const int32_t* sizes,
                                   const int64_t* nnz_off, const int32_t* idx, const float* vals, const float* B,
                                   int64_t ldb, float* C, int64_t ldc, int32_t max_rows, int32_t smem_optin,
                                   cudaStream_t s);
cudaError_t launch_transpose_csr(int32_t batch, const int64_t* row_off, const int32_t* sizes, const int32_t* row_ptr,
                                 const int32_t* col, const float* vals, int32_t* rowT, int32_t* colT, float* valsT,
                                 int32_t max_rows_hint, int64_t max_nnz_hint, int32_t num_sms, cudaStream_t s);
cudaError_t launch_sddmm(int32_t batch, int32_t k, const int64_t* row_off, const int32_t* sizes,
                         const int32_t* row_ptr, const int32_t* col, const float* B, int64_t ldb, const float* G,
                         int64_t ldg, float* out, int32_t max_rows_hint, int64_t max_nnz_hint, int32_t num_sms,
                         int32_t dbg, cudaStream_t s);
// fused backward (both adjoints) for streaming batches; *used = false when the
// shape / hints do not qualify (the caller then runs the separate kernels)
cudaError_t launch_backward_fused(int32_t batch, int32_t k, const int64_t* row_off, const int32_t* sizes,
                                  const int32_t* row_ptr, const int32_t* col, const float* vals, const float* B,
                                  int64_t ldb, const float* G, int64_t ldg, float* gB, int64_t ldgb, float* gvals,
                                  int32_t max_rows_hint, int64_t max_nnz_hint, int32_t num_sms, int32_t dbg,
                                  cudaStream_t s, bool* used);
cudaError_t launch_validate_csr(int32_t batch, const int64_t* row_off, const int32_t* sizes,
                                const int32_t* row_ptr, const int32_t* col, int* flag, cudaStream_t s);
cudaError_t launch_validate_coo(int32_t batch, const int64_t* row_off, const int32_t* sizes,
                                const int64_t* nnz_off, const int32_t* idx, int* flag, cudaStream_t s);
cudaError_t launch_validate_sizes(int32_t batch, const int32_t* sizes, int* flag, cudaStream_t s);

}  // namespace bspmm

struct bspmm_handle_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  unsigned flags = 0;
  int num_sms = 148;
  int smem_optin = 232448;
  int32_t hint_rows = 0;
  int64_t hint_nnz = 0;
  int32_t tune_kt = 0, tune_warps = 0, tune_ctas = 0, tune_chunks = 0;
  int32_t tune_tile_cb = 0;  // bspmm_set_tile_cb: tile kernel column block (0 = planner)
  bspmm_plan_t last_plan{};
  unsigned long long* trace = nullptr;  // debug: per-CTA phase timestamps
  int32_t dbg = 0;                      // debug bits: 1 = skip C stores
  // cached 2-D TMA descriptors (key: B, k, ldb, kt)
  bspmm::TmaMaps maps{};
  const void* maps_B = nullptr;
  int64_t maps_ldb = 0;
  int32_t maps_k = 0, maps_kt = 0;
  bool maps_ok = false;
  void* gcn_ws = nullptr;  // GCN layer: K-major split W, tile table, packed X
  int32_t gcn_math = 0;    // bspmm_set_gcn_math: 0 fp32 (3xTF32), 1 TF32, 2 BF16-rounded operands
  size_t gcn_ws_bytes = 0;
  int64_t launches = 0;
  std::string err;
  // device workspace (grown on demand)
  void* ws = nullptr;
  size_t ws_bytes = 0;
  int* dev_flag = nullptr;
  bool coo_fused_pending = false;  // a fused bspmm_coo ran since the last bspmm_sync
  unsigned long long* dev_sched = nullptr;  // dynamic-schedule ticket counter (zeroed once)
  // offsets scan state: [ticket u64][flags u32 x cap][agg i64 x cap][incl i64 x cap]
  void* scan_ws = nullptr;
  int32_t scan_cap = 0;
  uint32_t scan_epoch = 0;
  // e2e host-path buffers and streams
  void* hbuf = nullptr;
  size_t hbuf_bytes = 0;
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  // backward: the transpose runs on s_aux concurrently with the SDDMM (forked
  // from and joined back into `stream` within the call)
  cudaStream_t s_aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_handoff = nullptr;  // bspmm_set_stream: new stream waits for the old one
  cudaEvent_t ev[64] = {};
  bool in_backward = false;  // csr_backward's grad_B SpMM is running (no pre-wait prefetch)
};
