/*
 * bspmm_debug.h — experiment and diagnostics knobs of libbspmm.so.
 *
 * NOT part of the Batched SpMM contract (include/bspmm.h).  These entry points
 * exist for the measurement tools (tools/kbench.py sweeps, tools/trace.py
 * phase timelines) and for tests that pin every kernel variant to the same
 * bits; some settings make results undefined (debug bit 1).  Production
 * callers never need them: the defaults are what bspmm.h documents.
 */
#ifndef BSPMM_DEBUG_H_
#define BSPMM_DEBUG_H_

#include "bspmm.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Tuning override for experiments: kt (multiple of 4 on the vec path, 0 =
 * auto), consumer warps per CTA (0 = auto, <= 16; 15 with 4 chunks), CTAs per SM (0 = auto,
 * <= 4), column chunks per lane (0 = auto, <= 4). */
BSPMM_API bspmm_status_t bspmm_set_tuning(bspmm_handle_t h, int32_t kt, int32_t consumer_warps,
                                          int32_t ctas_per_sm, int32_t chunks);

/* Debug: per-CTA phase timestamps (%globaltimer, ns) of subsequent SpMM
 * launches are written to dev_buf [grid x 32] uint64 (slots: entry, after the
 * programmatic-launch wait, producer has unit-0 offsets, producer has unit-0
 * structure, producer done, first consumer warp sees unit 0, first consumer
 * warp done, CTA exit, first consumer warp done with unit 0; 9-15 and 16-27
 * producer issue steps of the first units, see spmm_csr.cu).  NULL disables
 * (the default). */
BSPMM_API bspmm_status_t bspmm_set_trace(bspmm_handle_t h, uint64_t* dev_buf);

/* Debug: timing-experiment bits for subsequent SpMM launches.  1 = compute but
 * do not store C (the result is then undefined); 2 = compute every unit from
 * global memory (no staging); 4 = no early B tile for the first unit of a
 * CTA; 8 = consumers repeat each unit's work 4 times;
 * 16 = no TMA-descriptor prefetch in the tile kernel; 32 = always copy
 * the CSR slice with TMA; 64 = force the static unit schedule; 128 = force the
 * dynamic one; 256 = SDDMM by the standalone kernel instead of the SpMM
 * pipeline's SDDMM mode; 512 = standalone SDDMM without the L2 prefetch of
 * the next matrix's B_i; 1024 = the SDDMM mode also for streaming batches,
 * and no one-unit consumer fast path in the SpMM (consumers wait for the
 * producer's header and CSR slice); 2048 = backward entirely on the
 * caller's stream (no auxiliary stream); 4096 = backward with only the
 * transpose on the auxiliary stream (grad_B SpMM on the caller's stream);
 * 8192 = GCN layer with one batched GEMM before the channel SpMMs instead
 * of channel GEMMs pipelined on the auxiliary stream; 16384 = never the
 * small-batch tile kernel (small batches run the pipeline kernel); 32768 =
 * tile kernel stages B by 16-byte cp.async everywhere (default: 2-D tensor
 * TMA for column blocks of >= 8 float4); 65536 = tile
 * kernel issues its row-pointer round trip after the B tile; 131072 = GCN
 * layer without the Z arithmetic, 262144 = GCN layer without the MMAs (both
 * leave Y undefined; timing only); 524288 = GCN layer with two groups of
 * Z-producer warps instead of three (3xTF32: three instead of two);
 * bits 20-21 = GCN feature-tile width (1: 64, 2: 128, 3: 256; 0: planner);
 * bit 22 (4194304) = GCN layer on CTA pairs (cta_group::2) regardless of the
 * planner, bit 23 (8388608) = GCN layer on single CTAs; bit 24 (16777216)
 * = SpMM kernels (tile and pipeline) without the pre-wait L2 prefetch of B
 * and the matrices' structure; bit 25 (33554432) =
 * that prefetch without the structure; bit 26 (67108864) = without the
 * CSR (col, val) run (default: B, the row-pointer slice and the (col, val)
 * run; SparseTensor input: B and the (idx, val) slice); bit 27 (134217728) = standalone SDDMM
 * reading the CSR structure from global memory (the round-1 kernel) instead
 * of the double-buffered shared stage; bit 28 (268435456) = standalone SDDMM
 * prefetching two grad_C rows ahead instead of one (k = 256).  0 (default) = normal. */
BSPMM_API bspmm_status_t bspmm_set_debug(bspmm_handle_t h, int32_t bits);

/* Small-batch tile kernel (spmm_tile.cu): float4 columns per tile (1, 2, 4,
 * 8, 16 or 32; rounded up to a power of two), 0 = the planner's choice.  A
 * non-zero value also lifts the one-wave eligibility limit. */
BSPMM_API bspmm_status_t bspmm_set_tile_cb(bspmm_handle_t h, int32_t cb);

#ifdef __cplusplus
}
#endif
#endif /* BSPMM_DEBUG_H_ */
