// plan.cpp — the launch planner (hot-path row a-3).
//
// PAPER.md:240-264 decides, from the matrix sizes, whether column cache
// blocking is applied (p column blocks, :257, :263) and how many threads each
// SpMM gets (subWarp * m_A for CSR, :259).  Re-derived for sm_100a:
//  * a unit is (matrix i, k-tile t); tiles = p = ceil(k / kt);
//  * kt starts at the whole row (capped at 512 columns on the float4 path,
//    128 on the scalar path) and is halved while the batch leaves more than
//    half the SMs idle (the paper's "batch 50 fails to fill the SMs", :377)
//    or a two-stage shared-memory ring of n_max x kt tiles does not fit;
//  * lanes per row = the paper's subWarp rule (:150-155) applied to the
//    tile's columns in per-lane chunks (float4 chunks on the vec path);
//  * persistent grid = min(units, SMs x CTAs/SM); each CTA walks units
//    blockIdx.x, +grid, ... through an S-stage TMA ring.
#include <algorithm>

#include "internal.h"

extern "C" BSPMM_API int32_t bspmm_subwarp(int32_t n_B) {
  if (n_B < 1) return 0;
  if (n_B > 16) return 32;
  return bspmm::pow2_ceil(n_B);
}

namespace bspmm {

bspmm_status_t make_plan(int32_t k, int32_t batch, bool vec, int32_t max_rows, int64_t max_nnz,
                         int32_t num_sms, int32_t smem_per_cta, int32_t kt_override, int32_t warps,
                         int32_t ctas_per_sm, int32_t chunks_pref, bspmm_plan_t* out, bool coo) {
  if (!out || k < 1 || batch < 0 || num_sms < 1 || smem_per_cta < 1024) return BSPMM_ERROR_INVALID_VALUE;
  bspmm_plan_t p{};
  const int32_t R = max_rows > 0 ? max_rows : kDefaultRows;
  const int64_t Z = max_nnz > 0 ? max_nnz : 8LL * R;
  const int32_t kmax = vec ? kMaxVecKt : kMaxScalarKt;
  const int32_t quantum = vec ? 4 : 1;

  int32_t kt;
  if (kt_override > 0) {
    kt = std::min(kt_override, kmax);
    if (vec) kt = align_up(kt, 4);
    kt = std::min(kt, align_up(k, quantum));
  } else {
    // column blocking only while the batch leaves more than half the SMs idle
    // AND the units are big: a CTA's units are issued one after another by
    // its producer (~1 us each on a cold start, tools/trace.py), so several
    // small units per CTA cost more than idle SMs (C4: kt 512 / 100 units 8.2
    // us, 256 / 200 8.7, 128 / 400 9.1 -- tools/kbench.py --sweep)
    kt = std::min(align_up(k, quantum), kmax);
    while (2LL * batch * ceil_div(k, kt) < num_sms && (int64_t)R * kt * 4 > 32768 && kt > 32)
      kt = align_up(kt / 2, quantum);
  }
  // CTAs per SM: one by default (sweeps: 2 never won once the consumers cover
  // several rows per warp); the knob stays for experiments
  int32_t ctas = ctas_per_sm > 0 ? ctas_per_sm : 1;
  // per-CTA shared-memory budget (B200: 228 KB per SM, 227 KB opt-in per CTA; 1 KB reserved per CTA)
  auto budget_for = [&](int32_t c) { return std::min(smem_per_cta, (233472 / c) - 1024); };
  // structure capacity: (col, val) pairs + row pointer
  // (stage regions are 128-byte aligned: 2-D TMA destinations)
  // CSR slice: col, vals, row pointers, each 16 + 4*count bytes rounded to 16 (spmm_csr.cu slice_bytes)
  const int64_t Zc = std::min<int64_t>(Z, 1 << 20);
  auto a16 = [](int64_t x) { return (x + 15) / 16 * 16; };
  int64_t s_need = 2 * a16(16 + 4 * Zc) + a16(16 + 4 * (R + 1));
  if (coo)  // fused COO mode (spmm_csr.cu coo_stage_bytes): + raw pairs, raw values, slots, row counters
    s_need = a16(s_need) + a16(8 * (Zc + 1)) + a16(4 * (Zc + 3)) + a16(4 * Zc) + a16(4 * (R + 1));
  int64_t s_bytes64 = align_up((int32_t)s_need, 128);
  auto stages_in = [&](int32_t kt_, int32_t budget_) {
    int64_t b = align_up(std::max<int32_t>(16, R * kt_ * 4), 128);
    int64_t per = b + s_bytes64;
    int64_t s = 0;
    while (s < kMaxStages && ring_prefix_bytes((int32_t)(s + 1)) + (s + 1) * per <= budget_) ++s;
    return (int32_t)s;
  };
  if (kt_override <= 0)
    while (stages_in(kt, budget_for(1)) < 2 && kt > quantum * 8) kt = align_up(kt / 2, quantum);
  const int32_t budget = budget_for(ctas);
  auto stages_for = [&](int32_t kt_) { return stages_in(kt_, budget); };

  int32_t stages = stages_for(kt);
  int32_t b_bytes = align_up(std::max<int32_t>(16, R * kt * 4), 128);
  int32_t s_bytes = (int32_t)s_bytes64;
  if (stages < 1) {
    // even one stage does not fit: shrink capacities; bigger matrices go direct
    s_bytes = std::min<int32_t>(s_bytes, budget / 4) / 128 * 128;
    b_bytes = (budget - ring_prefix_bytes(1) - s_bytes) / 128 * 128;
    stages = 1;
  }
  p.kt = kt;
  p.tiles = (int32_t)ceil_div(k, kt);
  p.vec = vec ? 1 : 0;
  // lanes per row: the paper's subWarp rule applied to the
  // tile's columns grouped in chunks of `pref` per lane (float4 chunks on the
  // vec path): one warp covers 32 / lanes rows per instruction
  const int32_t cols = vec ? (kt + 3) / 4 : kt;
  // 4 chunks per lane (4x more rows per warp instruction) pays off for small,
  // latency-bound batches with wide tiles (C4: 8.5 vs 9.7 us); large batches
  // prefer 2 (C5: 851 vs 860 us) -- tools/kbench.py sweeps
  const int64_t units_ = (int64_t)batch * ceil_div(k, kt);
  const int32_t pref_auto = (vec && kt >= 128 && units_ <= 4LL * num_sms) ? 4 : kDefaultChunks;
  const int32_t pref = chunks_pref > 0 ? std::min(chunks_pref, 4) : pref_auto;
  p.lanes = bspmm_subwarp((int32_t)ceil_div(cols, pref));
  const int32_t ch = (int32_t)ceil_div(cols, p.lanes);
  p.chunks = ch <= 1 ? 1 : (ch <= 2 ? 2 : 4);
  // consumer warps: 16 (544-thread CTA) up to 2 chunks per lane, 15 with 4
  const int32_t wmax = p.chunks >= 4 ? 15 : 16;
  const int32_t W = coo ? coo_consumer_warps(warps) : warps > 0 ? std::min(warps, wmax) : wmax;
  p.stages = stages;
  p.stage_b_bytes = b_bytes;
  p.stage_s_bytes = s_bytes;
  p.smem_bytes = ring_prefix_bytes(stages) + stages * (b_bytes + s_bytes);
  p.threads = coo ? 32 * kCooWarps : 32 * (1 + W);
  p.units = (int64_t)batch * p.tiles;
  p.grid = (int32_t)std::min<int64_t>(p.units, (int64_t)num_sms * ctas);
  p.max_rows = R;
  // static round-robin schedule by default: the dynamic one (global ticket
  // counter, debug bit 128) measured slower on C3/C4 (13.0 vs 12.1 us, 10.1 vs
  // 9.0 us) because its per-unit ticket -> metadata chain is serial in the
  // producer; it is kept for experiments
  p.sched = 0;
  *out = p;
  return BSPMM_SUCCESS;
}

}  // namespace bspmm

extern "C" BSPMM_API bspmm_status_t bspmm_plan(int32_t k, int32_t batch, int32_t aligned, int32_t max_rows,
                                               int64_t max_nnz, int32_t num_sms, int32_t smem_per_cta,
                                               int32_t kt_override, int32_t consumer_warps,
                                               int32_t ctas_per_sm, int32_t chunks, bspmm_plan_t* out) {
  return bspmm::make_plan(k, batch, aligned != 0, max_rows, max_nnz, num_sms, smem_per_cta, kt_override,
                          consumer_warps, ctas_per_sm, chunks, out);
}
