/*
 * bspmm.h — C ABI of the B200-native Batched SpMM library (libbspmm.so).
 *
 * The operation (§IV, "Batched Algorithm for SpMM", lines 240-264,
 * and the GCN use of it, Fig. algo:graph_conv_batched, lines 304-321):
 * for every matrix i of a mini-batch, in ONE launch,
 *
 *     C_i = A_i * B_i          ("SpMM computes C = AB")
 *
 * with A_i an n_i x n_i sparse adjacency matrix (square; graph
 * convention a_uu = 1, a_vu = 1 for an edge u->v) stored as CSR
 * (rpt / colids / values, Fig. algo:code_swa_spmm_csr :196-207)
 * or as a TF SparseTensor (interleaved (row, col) index pairs + values,
 * PAPER.md:74, Fig. algo:code_swa_spmm_st :175-185, entries unsorted :141),
 * and B_i / C_i dense n_i x k fp32 row-major (PAPER.md:101 C[rid][j]); k is
 * uniform across the batch.
 *
 * Batch layout (the "reshape to (m_X * batchsize) x n_X"):
 * the dense rows of all matrices are concatenated.  Matrix i owns the global
 * rows [row_off[i], row_off[i] + n_i) of B and C.  row_off replaces the
 * paper's host-built pointer arrays; it is int64.
 *
 * Conventions (every entry point):
 *  - All functions return bspmm_status_t; nothing is thrown across the ABI.
 *  - Pointers marked "dev" are device pointers on the handle's device, owned
 *    by the caller (typically torch tensors); "host" pointers are host memory.
 *    The library never frees caller memory.  The handle owns its device
 *    workspace (grown on demand, freed by bspmm_destroy), one internal
 *    non-blocking auxiliary stream and its events (created with the handle, so
 *    calls can be captured into a CUDA graph on first use), and BORROWS the
 *    stream given to bspmm_create / bspmm_set_stream.  bspmm_csr_backward
 *    forks work onto the auxiliary stream and joins it back into the caller's
 *    stream before returning (also on error), so to the caller every call is
 *    ordered on its stream.
 *  - Handle state (workspace, scan state, error flag) is shared by the calls
 *    of a handle: when bspmm_set_stream changes the stream, the new stream is
 *    made to wait for all work enqueued so far on the previous one (the
 *    previous stream must still exist at that point).
 *  - Calls on device pointers are asynchronous on the handle's stream: they
 *    enqueue kernels and return.  Inputs must stay alive and unmodified until
 *    the stream reaches that point.  Device faults surface from a later call,
 *    bspmm_sync or bspmm_destroy (BSPMM_ERROR_CUDA).
 *  - Host-side checks: NULL where required, batch < 0, k < 1, ld < k.
 *    With BSPMM_VALIDATE the library also checks every index/offset on the
 *    device and SYNCHRONISES at the end of the call to report
 *    BSPMM_ERROR_INDEX.  Without it, out-of-range indices are undefined
 *    behaviour (as in cuSPARSE).
 *  - Degenerate inputs are legal: batch = 0 is a no-op; n_i = 0 writes
 *    nothing; rows with no entries are written as +0.0 by the same kernel
 *    (the paper's "set matrix C to O", PAPER.md:95/:177/:198, without a
 *    separate initialisation launch).  C is OVERWRITTEN
 *    (no alpha/beta).  Rows between row_off[i] + n_i and row_off[i+1]
 *    (padding) are never touched.  Duplicate (row, col) entries are summed.
 *  - Fast path: k % 4 == 0, ldb % 4 == 0, ldc % 4 == 0 and 16-byte aligned
 *    B and C (float4 lanes, TMA bulk staging).  Anything else runs the scalar
 *    path; that is not an error.
 *  - A handle is not thread-safe; distinct handles are independent.
 *  - Multi-GPU: no ABI change on the hot path.  One handle per rank/device,
 *    called on the rank's contiguous sub-batch (bspmm_partition), offsets
 *    rebased to 0.  Optional reassembly of the full C on every GPU is fused
 *    into the store (bspmm_csr_multicast + the bspmm_mc_* team buffers).
 */
#ifndef BSPMM_H_
#define BSPMM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define BSPMM_API __attribute__((visibility("default")))
#else
#define BSPMM_API
#endif

typedef struct bspmm_handle_s* bspmm_handle_t;
typedef struct bspmm_mc_s* bspmm_mc_t; /* NVSwitch multicast team buffer (NEXT-4b) */

typedef enum {
  BSPMM_SUCCESS = 0,
  BSPMM_ERROR_INVALID_VALUE = 1, /* NULL where required, batch<0, k<1, ld<k, bad flags   */
  BSPMM_ERROR_OUT_OF_MEMORY = 2, /* workspace growth failed                              */
  BSPMM_ERROR_CUDA = 3,          /* CUDA API / launch / async error; see last_error_string */
  BSPMM_ERROR_INDEX = 4,         /* BSPMM_VALIDATE found an index or offset out of range  */
  BSPMM_ERROR_NOT_SUPPORTED = 5  /* device is not sm_100 (B200), or no device             */
} bspmm_status_t;

#define BSPMM_VALIDATE 0x1u /* device pass checking every index; synchronising; off by default */

/* Launch plan ("decides whether the cache blocking is
 * applied and how many threads are assigned"), re-derived for sm_100a: a unit
 * of work is (matrix i, k-tile t); persistent CTAs walk the units. */
typedef struct {
  int32_t kt;             /* k-tile width in columns (column cache blocking) */
  int32_t tiles;          /* p = ceil(k / kt) column blocks per matrix    */
  int32_t lanes;          /* lanes per row: subWarp rule on per-lane chunks  */
  int32_t vec;            /* 1: float4 lanes + TMA bulk staging; 0: scalar lanes + cp.async     */
  int32_t chunks;         /* float4 (vec) or float (scalar) column chunks per lane              */
  int32_t stages;         /* shared-memory ring depth per CTA                                   */
  int32_t stage_b_bytes;  /* B-tile capacity per stage (rows * kt * 4 must fit to be staged)    */
  int32_t stage_s_bytes;  /* sparse-structure capacity per stage (rpt + (col,val) pairs)        */
  int32_t smem_bytes;     /* dynamic shared memory per CTA                                      */
  int32_t threads;        /* CTA size: 1 producer warp + consumer warps                         */
  int32_t grid;           /* persistent CTAs launched                                           */
  int32_t max_rows;       /* planning assumption for max n_i (hint or default)                  */
  int32_t sched;          /* 0: static round-robin units; 1: dynamic (global ticket counter)    */
  int64_t units;          /* batch * tiles                                                      */
  int32_t kernel;         /* 0: persistent TMA-ring pipeline; 1: small-batch tile kernel (one   *
                           * CTA per (matrix, column block); kt = 4 * block, lanes = block;   *
                           * CSR and, in bspmm_coo, SparseTensor input)                        */
} bspmm_plan_t;

/* ---- lifetime -------------------------------------------------------- */

/* Creates a handle on `device` (cudaSetDevice is NOT left changed).  stream is
 * a cudaStream_t (NULL = legacy default stream), borrowed.  flags: 0 or
 * BSPMM_VALIDATE.  Errors: INVALID_VALUE (out NULL, bad flags),
 * NOT_SUPPORTED (no device / not compute capability 10.0), CUDA. */
BSPMM_API bspmm_status_t bspmm_create(bspmm_handle_t* out, int device, void* stream, unsigned flags);

/* Synchronises the handle's stream, frees the workspace.  NULL is a no-op. */
BSPMM_API bspmm_status_t bspmm_destroy(bspmm_handle_t h);

/* Re-targets the borrowed stream (e.g. torch's current stream per call).  On
 * a change, the new stream waits (one event) for everything already enqueued
 * on the old one, so work of this handle never overlaps across streams; the
 * wait is skipped while either stream is capturing a CUDA graph.  Errors:
 * INVALID_VALUE, CUDA. */
BSPMM_API bspmm_status_t bspmm_set_stream(bspmm_handle_t h, void* stream);

/* Planner hints (host scalars, optional; 0 = unknown).  max_rows: max n_i
 * in upcoming batches; max_nnz: max entries of one A_i.  Matrices larger than
 * the plan's stage capacity still run correctly, reading B from global memory
 * directly (the paper's "case 3"). */
BSPMM_API bspmm_status_t bspmm_set_hints(bspmm_handle_t h, int32_t max_rows, int64_t max_nnz);

/* Waits for all work enqueued by this handle; surfaces asynchronous errors. */
BSPMM_API bspmm_status_t bspmm_sync(bspmm_handle_t h);

/* ---- the hot path ---------------------------------------------------- */

/* Batched CSR SpMM (SWA SpMM for CSR, Fig.
 * algo:code_swa_spmm_csr; batched per PAPER.md:259-264):
 *   for i in [0, batch), r in [0, n_i), c in [0, k):
 *     C[(row_off[i]+r)*ldc + c] = sum_{e = row_ptr[g]}^{row_ptr[g+1]-1}
 *                                  vals[e] * B[(row_off[i]+col_idx[e])*ldb + c],
 *     g = row_off[i] + r, accumulated in fp32 FMA in storage order from +0.0.
 *  row_off  [batch+1] dev int64, or NULL: then `sizes` is required and the
 *           layout is packed; the library derives the offsets on the device
 *           (small batches: warp prefix sums inside the SpMM launch itself;
 *           large ones: the look-back scan kernel of bspmm_build_offsets).
 *  sizes    [batch]   dev int32 n_i, or NULL: n_i = row_off[i+1] - row_off[i].
 *  row_ptr  [row_off[batch]+1] dev int32: block-diagonal CSR row pointer
 *           holding ABSOLUTE positions into col_idx / vals.
 *  col_idx  [nnz] dev int32 LOCAL column ids, 0 <= c < n_i (square A_i).
 *  vals     [nnz] dev fp32.  col_idx / vals / B / C may be NULL only when they
 *           have no elements (no entries / no rows).
 *  B        [row_off[batch] x ldb] dev fp32 row-major, ldb >= k.
 *  C        same shape with ldc >= k; must not alias B.
 * Errors: INVALID_VALUE, CUDA, INDEX (VALIDATE only). */
BSPMM_API bspmm_status_t bspmm_csr(bspmm_handle_t h, int32_t batch, int32_t k, const int64_t* row_off,
                                   const int32_t* sizes, const int32_t* row_ptr, const int32_t* col_idx,
                                   const float* vals, const float* B, int64_t ldb, float* C, int64_t ldc);

/* bspmm_csr with the all-gather of C fused into the store (SURVEY §8(e)
 * optional reassembly, §8(f) NEXT-4b; the paper is single-GPU):
 * identical arithmetic and bits, but every C row is written with ONE
 * multimem.st to `C_mc`, an address inside the MULTICAST range of a team
 * buffer (bspmm_mc_bind), so it lands in the bound buffer of every GPU of the
 * team.  Rank r passes C_mc = mc_ptr + row_base_r * ldc * 4 bytes for its
 * shard (the shard's own offsets start at 0) and, after the call, a barrier
 * over the team (e.g. an NCCL all_reduce on the same stream) makes the full C
 * readable through each rank's UNICAST pointer.  The kernel ends with a
 * system-scope fence.  Same arguments and errors as bspmm_csr; C_mc must not
 * be an ordinary allocation (undefined behaviour). */
BSPMM_API bspmm_status_t bspmm_csr_multicast(bspmm_handle_t h, int32_t batch, int32_t k, const int64_t* row_off,
                                             const int32_t* sizes, const int32_t* row_ptr, const int32_t* col_idx,
                                             const float* vals, const float* B, int64_t ldb, float* C_mc,
                                             int64_t ldc);

/* ---- NVSwitch multicast team buffers (NEXT-4b) ------------------------ *
 * A team of num_devices GPUs (one process per GPU, or num_devices = 1) shares
 * one buffer of >= bytes (rounded up to the multicast granularity).
 * Protocol: the root calls bspmm_mc_create (exportable = 1 when num_devices >
 * 1: *fd_out receives a POSIX file descriptor the caller sends to the other
 * ranks, e.g. SCM_RIGHTS); every other rank calls bspmm_mc_import with it.
 * Both add the caller's `device` to the team.  After ALL members have joined
 * (a barrier), each calls bspmm_mc_bind: it allocates `bytes` on its device,
 * binds them and returns the unicast (own copy, ordinary loads/stores) and
 * multicast (stores reach every member) device pointers.  Barrier again
 * before the first multicast store.  bspmm_mc_destroy unmaps and frees (NULL
 * ok).  Errors: INVALID_VALUE, NOT_SUPPORTED (no NVSwitch multicast on this
 * device / driver), OUT_OF_MEMORY, CUDA.  The caller owns the fd. */
BSPMM_API int32_t bspmm_mc_supported(int device);
BSPMM_API bspmm_status_t bspmm_mc_create(int device, int num_devices, size_t bytes, int exportable,
                                         bspmm_mc_t* out, int* fd_out);
BSPMM_API bspmm_status_t bspmm_mc_import(int device, int num_devices, size_t bytes, int fd, bspmm_mc_t* out);
BSPMM_API bspmm_status_t bspmm_mc_bind(bspmm_mc_t mc, void** uc_ptr, void** mc_ptr);
BSPMM_API size_t bspmm_mc_bytes(bspmm_mc_t mc);
/* Which driver call failed last in this thread (bspmm_mc_* only). */
BSPMM_API const char* bspmm_mc_last_error(void);
BSPMM_API bspmm_status_t bspmm_mc_destroy(bspmm_mc_t mc);

/* Batched COO / SparseTensor SpMM (Fig.
 * algo:code_swa_spmm_st).  The entries of A_i are [nnz_off[i], nnz_off[i+1])
 * of idx / vals, in ANY order.  They are first converted on the device to
 * canonical CSR (stable by (row, col): duplicates keep their input order) and
 * then multiplied by the CSR kernel, so the result is deterministic (the
 * paper's atomic accumulation, is not).
 *  nnz_off     [batch+1] dev int64.
 *  idx         [nnz][2] dev int32: (row, col) LOCAL pairs, interleaved
 *              exactly as TF SparseTensor ids (rid = ids[2e],
 *              cid = ids[2e+1]).
 *  total_rows  host: row_off[batch] (sizes the CSR row pointer).
 *  total_nnz   host: nnz_off[batch].
 *  csr_*_out   dev, nullable as a group: when non-NULL the built CSR is
 *              written there ([total_rows+1], [total_nnz], [total_nnz]),
 *              otherwise into handle workspace.
 * row_off may be NULL (then built from sizes); nnz_off is required.
 * With planner hints set (bspmm_set_hints: max_rows, max_nnz bounding every
 * A_i), the fast path (k, ldb, ldc % 4 == 0, aligned B, C) and no csr_*_out,
 * the conversion is FUSED into the SpMM launch: each unit's SparseTensor slice
 * is staged and sorted into CSR in shared memory (same canonical order, same
 * bits) -- by converter warps of the persistent kernel, or, for batches whose
 * tiles are all resident at once, by each tile CTA of the small-batch kernel
 * while its B tile lands (bspmm_last_plan: kernel 0 / 1).  A matrix beyond
 * the hints is then skipped -- ITS ROWS OF C ARE NOT
 * WRITTEN -- and reported as BSPMM_ERROR_INVALID_VALUE by the next
 * bspmm_sync: callers that cannot guarantee the hints must call bspmm_sync
 * after the call (the Python binding's Handle.coo(checked=True) does). */
BSPMM_API bspmm_status_t bspmm_coo(bspmm_handle_t h, int32_t batch, int32_t k, const int64_t* row_off,
                                   const int32_t* sizes, const int64_t* nnz_off, const int32_t* idx,
                                   const float* vals, const float* B, int64_t ldb, float* C, int64_t ldc,
                                   int64_t total_rows, int64_t total_nnz, int32_t* csr_row_ptr_out,
                                   int32_t* csr_col_out, float* csr_val_out);

/* Arithmetic of the tensor-core GEMM in bspmm_gcn_layer (the SpMM part,
 * Z = A_ch X, is always fp32 FMA in storage order):
 *  BSPMM_GCN_FP32 (default) 3xTF32: both operands split into a TF32 head and
 *                 an fp32 remainder, three tcgen05 MMAs per step
 *                 (head.head + head.rem + rem.head): fp32-accurate;
 *  BSPMM_GCN_TF32 one MMA on the fp32 values (TF32 inputs, 10-bit mantissa);
 *  BSPMM_GCN_BF16 one MMA on operands rounded to BF16 (7-bit mantissa), run
 *                 on the TF32 datapath (BF16 values are exact in TF32).
 * Errors: INVALID_VALUE (unknown mode). */
#define BSPMM_GCN_FP32 0
#define BSPMM_GCN_TF32 1
#define BSPMM_GCN_BF16 2
BSPMM_API bspmm_status_t bspmm_set_gcn_math(bspmm_handle_t h, int32_t mode);

/* Fused batched graph-convolution layer (PAPER.md Fig. algo:graph_conv_batched,
 * :304-321; Eq. (2) :66-68):  Y = sum_ch A_ch (X W_ch + 1 bias_ch^T).
 *  X      [total_rows x ldx] dev fp32 (node features, stacked graphs; n_x used)
 *  W      [channels][n_x][k] dev fp32, dense contiguous
 *  bias   [channels][k] dev fp32, nullable (= 0)
 *  row_ptr [channels][total_rows + 1] dev int32: one block-diagonal CSR per
 *         channel (channel-specific adjacency), absolute positions into the
 *         shared col / vals arrays; col LOCAL ids.
 *  Y      [total_rows x ldy] dev fp32 (overwritten; padding rows untouched).
 * Computed as ONE tensor-core GEMM per 128-row x (<=128)-feature output tile
 * through the exact identity Y = [A_1 X | ... | A_C X | r_1..r_C] .
 * [W_1; ...; W_C; b_1^T; ...; b_C^T] (r_ch = rowsum A_ch): the left operand
 * is produced in shared memory by the SpMM row loop (never in HBM), the
 * channel sum and the bias are part of the TMEM accumulation (csrc/
 * gcn_fused.cu).  Two launches: a preparation kernel (W to K-major, split for
 * 3xTF32; tile table) and the fused kernel.  Handle workspace: 2 x k x
 * (channels * ceil32(n_x) + 32 ceil(channels/32)) floats + one int per 128
 * rows (+ a packed copy of X when ldx % 4 != 0 or X is not 16-byte aligned).
 * Errors: INVALID_VALUE, NOT_SUPPORTED (total_rows >= 2^31), CUDA, INDEX
 * (VALIDATE). */
BSPMM_API bspmm_status_t bspmm_gcn_layer(bspmm_handle_t h, int32_t batch, int32_t channels, int32_t n_x, int32_t k,
                                         const int64_t* row_off, const int32_t* sizes, const int32_t* row_ptr,
                                         const int32_t* col, const float* vals, const float* X, int64_t ldx,
                                         const float* W, const float* bias, float* Y, int64_t ldy,
                                         int64_t total_rows);

/* The paper's own SWA SpMM for SparseTensor (Fig.
 * algo:code_swa_spmm_st, output tile in shared memory per Fig.
 * batched_spmm_algo (a)/(b)): one thread block per (matrix, column block), a
 * sub-warp per nonzero, atomic accumulation into the shared C tile; matrices
 * above the tile capacity accumulate with global atomics (case 3,
 * PAPER.md:249-252).  Same arguments and result as bspmm_coo (C overwritten)
 * but the summation order is NOT deterministic (results agree within the
 * north_star bound, not bitwise).  Requires k, ldb, ldc % 4 == 0 and 16-byte
 * aligned B, C (else BSPMM_ERROR_NOT_SUPPORTED).  Planner hint max_rows sizes
 * the shared tile. */
BSPMM_API bspmm_status_t bspmm_coo_atomic(bspmm_handle_t h, int32_t batch, int32_t k, const int64_t* row_off,
                                          const int32_t* sizes, const int64_t* nnz_off, const int32_t* idx,
                                          const float* vals, const float* B, int64_t ldb, float* C, int64_t ldc);

/* COO -> CSR alone (hot-path row a-2; exported for the bit-exact tests).
 * Output order per matrix: by (row, col, original position); row_ptr holds
 * absolute positions (nnz_off[i] + local); padding rows between matrices get
 * empty ranges; row_ptr[row_off[batch]] = nnz_off[batch].  vals are moved
 * bitwise.  row_off must be given (dev int64). */
BSPMM_API bspmm_status_t bspmm_coo2csr(bspmm_handle_t h, int32_t batch, const int64_t* row_off,
                                       const int32_t* sizes, const int64_t* nnz_off, const int32_t* idx,
                                       const float* vals, int64_t total_rows, int64_t total_nnz,
                                       int32_t* row_ptr_out, int32_t* col_out, float* val_out);

/* Batch-offset builder (hot-path row a-1): offsets_out[0] = 0,
 * offsets_out[i+1] = offsets_out[i] + sizes[i], int64, on the device
 * (replaces the host pointer arrays + H2D copy of PAPER.md:281/:343).
 * sizes [batch] dev int32, offsets_out [batch+1] dev int64. */
BSPMM_API bspmm_status_t bspmm_build_offsets(bspmm_handle_t h, int32_t batch, const int32_t* sizes,
                                             int64_t* offsets_out);

/* ---- backward ("also applied to backward propagation") ------
 * For C_i = A_i B_i and an upstream gradient G = dL/dC (layout of C), the
 * standard adjoints: dL/dB_i = A_i^T G_i and dL/dval_e = <G[row_e], B[col_e]>. */

/* Per-matrix transpose of a block-diagonal CSR: A_i^T in canonical (row, col,
 * original position) order, absolute row pointers, LOCAL column ids, values
 * moved bitwise.  row_off (dev) required; outputs [total_rows+1],
 * [total_nnz], [total_nnz] dev.  A static graph can be transposed once and
 * then multiplied with bspmm_csr. */
BSPMM_API bspmm_status_t bspmm_csr_transpose(bspmm_handle_t h, int32_t batch, const int64_t* row_off,
                                             const int32_t* sizes, const int32_t* row_ptr, const int32_t* col,
                                             const float* vals, int64_t total_rows, int64_t total_nnz,
                                             int32_t* rowT_out, int32_t* colT_out, float* valsT_out);

/* Batched SDDMM at A's pattern: out[e] = sum_{c<k} G[row_e][c] * B[col_e][c]
 * for every stored entry e (fp32, deterministic warp-shuffle reduction;
 * accurate to the fp32 dot-product bound).  out [nnz] dev. */
BSPMM_API bspmm_status_t bspmm_sddmm(bspmm_handle_t h, int32_t batch, int32_t k, const int64_t* row_off,
                                     const int32_t* sizes, const int32_t* row_ptr, const int32_t* col, const float* B,
                                     int64_t ldb, const float* G, int64_t ldg, float* out);

/* Backward of bspmm_csr: grad_B (nullable) = A^T grad_C (bitwise the fp32
 * storage-order sum over the canonical A^T); grad_vals (nullable) =
 * SDDMM(grad_C, B).  With both requested on a streaming batch (more than 8
 * matrices per SM, planner hints set, k <= 256, 16-byte aligned rows) one
 * fused kernel computes both from grad_C staged once per matrix, forming
 * A_i^T in shared memory; otherwise an internal transpose + the forward
 * kernel, and the SDDMM.  Both give the same bits.  grad_B must not alias
 * grad_C.  total_rows / total_nnz: host sizes of the CSR. */
BSPMM_API bspmm_status_t bspmm_csr_backward(bspmm_handle_t h, int32_t batch, int32_t k, const int64_t* row_off,
                                            const int32_t* sizes, const int32_t* row_ptr, const int32_t* col,
                                            const float* vals, const float* B, int64_t ldb, const float* grad_C,
                                            int64_t ldgc, float* grad_B, int64_t ldgb, float* grad_vals,
                                            int64_t total_rows, int64_t total_nnz);

/* End-to-end call on HOST buffers (packed layout, ldb = ldc = k): copies the
 * inputs host->device (pinned memory recommended), builds offsets, runs the
 * CSR kernel and copies C back, pipelined in row chunks across copy and
 * compute streams; returns when C_host is complete (synchronous).
 *  sizes_host [batch], row_ptr_host [total_rows+1] (absolute),
 *  col_host / vals_host [total_nnz], B_host / C_host [total_rows x k]. */
BSPMM_API bspmm_status_t bspmm_csr_host(bspmm_handle_t h, int32_t batch, int32_t k, const int32_t* sizes_host,
                                        const int32_t* row_ptr_host, const int32_t* col_host,
                                        const float* vals_host, const float* B_host, float* C_host,
                                        int64_t total_rows, int64_t total_nnz);

/* ---- host-only helpers (no device needed) ----------------------------- */

/* Multi-GPU partition (hot-path row a-7): contiguous graph ranges balanced
 * by cost c_i = nnz_i * k.  With P_j = sum_{i<j} c_i and T = P_batch:
 * split[0] = 0, split[parts] = batch, and for 0 < r < parts split[r] is the
 * smallest j in [0, batch] with P_j * parts >= r * T (if T == 0,
 * floor(r * batch / parts)).  Rank r owns graphs [split[r], split[r+1]).
 * nnz_off [batch+1] HOST int64; split_out [parts+1] HOST int32. */
BSPMM_API bspmm_status_t bspmm_partition(int32_t batch, const int64_t* nnz_off, int32_t k, int32_t parts,
                                         int32_t* split_out);

/* The paper's subWarp rule: 32 if n_B > 16, else the
 * smallest power of two >= n_B.  Returns 0 for n_B < 1. */
BSPMM_API int32_t bspmm_subwarp(int32_t n_B);

/* The launch plan bspmm_csr would use for (k, batch, aligned) on a device
 * with `num_sms` SMs and `smem_per_cta` bytes of opt-in shared memory
 * (max_rows / max_nnz: hints, 0 = unknown; kt_override / warps / ctas_per_sm /
 * chunks: tuning, 0 = auto).  Pure host function. */
BSPMM_API bspmm_status_t bspmm_plan(int32_t k, int32_t batch, int32_t aligned, int32_t max_rows, int64_t max_nnz,
                                    int32_t num_sms, int32_t smem_per_cta, int32_t kt_override,
                                    int32_t consumer_warps, int32_t ctas_per_sm, int32_t chunks,
                                    bspmm_plan_t* out);

/* The plan used by the most recent bspmm_csr / bspmm_coo on this handle. */
BSPMM_API bspmm_status_t bspmm_last_plan(bspmm_handle_t h, bspmm_plan_t* out);

/* Kernel launches issued by this handle since creation (for bench claims). */
BSPMM_API int64_t bspmm_launch_count(bspmm_handle_t h);

BSPMM_API const char* bspmm_status_string(bspmm_status_t s);
BSPMM_API const char* bspmm_last_error_string(bspmm_handle_t h);

#ifdef __cplusplus
}
#endif
#endif /* BSPMM_H_ */
