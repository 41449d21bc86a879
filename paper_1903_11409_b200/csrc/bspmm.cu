// bspmm.cu — the C ABI (include/bspmm.h): handle, validation, workspace,
// planning and launches; plus the end-to-end host-buffer path.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <new>
#include <string>

#include <cudaTypedefs.h>

#include "internal.h"

using namespace bspmm;

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

bspmm_status_t fail_cuda(bspmm_handle_t h, cudaError_t e, const char* where) {
  if (h) h->err = std::string(where) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? BSPMM_ERROR_OUT_OF_MEMORY : BSPMM_ERROR_CUDA;
}
bspmm_status_t fail(bspmm_handle_t h, bspmm_status_t s, const char* msg) {
  if (h) h->err = msg;
  return s;
}

#define CK(h, expr)                                        \
  do {                                                     \
    cudaError_t e_ = (expr);                               \
    if (e_ != cudaSuccess) return fail_cuda(h, e_, #expr); \
  } while (0)

inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

// every stream that may still use handle-owned device memory
cudaError_t sync_streams(bspmm_handle_t h) {
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e == cudaSuccess && h->s_aux) e = cudaStreamSynchronize(h->s_aux);
  if (e == cudaSuccess && h->s_h2d) e = cudaStreamSynchronize(h->s_h2d);
  if (e == cudaSuccess && h->s_d2h) e = cudaStreamSynchronize(h->s_d2h);
  return e;
}

// grow a device buffer (synchronises the handle's streams before freeing)
bspmm_status_t grow(bspmm_handle_t h, void** buf, size_t* cap, size_t need) {
  if (need <= *cap) return BSPMM_SUCCESS;
  if (*buf) {
    CK(h, sync_streams(h));
    CK(h, cudaFree(*buf));
    *buf = nullptr;
    *cap = 0;
  }
  size_t sz = al256(std::max(need, *cap + *cap / 2));
  CK(h, cudaMalloc(buf, sz));
  *cap = sz;
  return BSPMM_SUCCESS;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bspmm_status_t check_validate_flag(bspmm_handle_t h) {
  int host = 0;
  CK(h, cudaMemcpyAsync(&host, h->dev_flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  if (host) {
    h->err = "BSPMM_VALIDATE: index/offset out of range (flag " + std::to_string(host) + ")";
    return BSPMM_ERROR_INDEX;
  }
  return BSPMM_SUCCESS;
}

// persistent look-back scan workspace: grown on demand, zeroed once; epochs tag each call
bspmm_status_t scan_state(bspmm_handle_t h, int32_t batch, ScanState* ss) {
  const int32_t tiles = std::max<int32_t>(1, scan_tiles(batch));
  if (tiles > h->scan_cap) {
    const int32_t cap = std::max<int32_t>(tiles, 64);
    const size_t bytes = 256 + al256((size_t)cap * 4) + 2 * al256((size_t)cap * 8);
    if (h->scan_ws) {
      CK(h, sync_streams(h));
      CK(h, cudaFree(h->scan_ws));
      h->scan_ws = nullptr;
      h->scan_cap = 0;
    }
    CK(h, cudaMalloc(&h->scan_ws, bytes));
    CK(h, cudaMemsetAsync(h->scan_ws, 0, bytes, h->stream));
    h->scan_cap = cap;
    h->scan_epoch = 0;
  }
  char* b = static_cast<char*>(h->scan_ws);
  if (++h->scan_epoch >= (1u << 30)) {  // epoch wrap: clear the status words once
    CK(h, cudaMemsetAsync(b + 256, 0, (size_t)h->scan_cap * 4, h->stream));
    h->scan_epoch = 1;
  }
  ss->ticket = reinterpret_cast<unsigned long long*>(b);
  ss->flags = reinterpret_cast<uint32_t*>(b + 256);
  ss->agg = reinterpret_cast<int64_t*>(b + 256 + al256((size_t)h->scan_cap * 4));
  ss->incl = ss->agg + al256((size_t)h->scan_cap * 8) / 8;
  ss->epoch = h->scan_epoch;
  return BSPMM_SUCCESS;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// link-time libcuda dependency)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      return nullptr;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  return encode;
}

// 2-D fp32 tensor map: `outer` rows of `inner` elements, row pitch `pitch_bytes`
bool encode_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t pitch_bytes,
               uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swizzle) {
  PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
  if (!encode) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  const cuuint64_t strides[1] = {(cuuint64_t)pitch_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D TMA descriptors for the k-tiled staging path, cached per (B, k, ldb, kt).
// Encoded with the driver's cuTensorMapEncodeTiled, fetched through the runtime
// (no link-time libcuda dependency).  Returns nullptr when not applicable.
const TmaMaps* tma_maps(bspmm_handle_t h, const float* B, int32_t k, int64_t ldb, int32_t kt) {
  if (kt % 32 != 0 || kt > 256 || ldb == kt) return nullptr;
  if (h->maps_ok && h->maps_B == B && h->maps_k == k && h->maps_ldb == ldb && h->maps_kt == kt) return &h->maps;
  PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
  if (!encode) return nullptr;
  const cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)0x7fffffff};  // rows: never read out of range
  const cuuint64_t strides[1] = {(cuuint64_t)ldb * 4};
  const cuuint32_t estr[2] = {1, 1};
  for (int b = 0; b < kTmaMaps; ++b) {
    const cuuint32_t box[2] = {(cuuint32_t)kt, (cuuint32_t)(1u << b)};
    CUresult r = encode(&h->maps.m[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(B), dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      h->maps_ok = false;
      return nullptr;
    }
  }
  h->maps_B = B;
  h->maps_k = k;
  h->maps_ldb = ldb;
  h->maps_kt = kt;
  h->maps_ok = true;
  return &h->maps;
}

bspmm_status_t plan_for(bspmm_handle_t h, int32_t batch, int32_t k, bool aligned, bspmm_plan_t* plan) {
  bspmm_status_t st = make_plan(k, batch, aligned, h->hint_rows, h->hint_nnz, h->num_sms, h->smem_optin,
                                h->tune_kt, h->tune_warps, h->tune_ctas, h->tune_chunks, plan);
  if (st != BSPMM_SUCCESS) return fail(h, st, "planner rejected the arguments");
  h->last_plan = *plan;
  return BSPMM_SUCCESS;
}

}  // namespace

// the pre-wait L2 prefetch applies to this call (not under debug bit 24, and
// not for the grad_B SpMM inside csr_backward: its structure is the
// transpose's output, written by the kernel right before -- the racy reads
// would only see stale values, and the prefetch measured slower there: C2
// backward 9.5 vs 8.6 us)
static inline bool prewait_prefetch(bspmm_handle_t h) { return !(h->dbg & kDbgNoPrewaitPrefetch) && !h->in_backward; }

// The device allocation containing p (cuMemGetAddressRange through the
// runtime's driver entry point): the kernels' pre-wait L2 prefetch clips its
// (possibly stale) addresses to it.  Queried on every call -- a cached range
// could outlive its allocation (freed, and a smaller one placed at the same
// base) and let a prefetch reach unmapped memory.
bool bspmm::alloc_range(bspmm_handle_t h, const void* p, uint64_t* lo, uint64_t* hi) {
  (void)h;
  static const PFN_cuMemGetAddressRange_v3020 range = []() -> PFN_cuMemGetAddressRange_v3020 {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess && fn)
      return reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
    cudaGetLastError();
    return nullptr;
  }();
  if (!range || !p) return false;
  CUdeviceptr base = 0;
  size_t bytes = 0;
  if (range(&base, &bytes, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS || bytes == 0) return false;
  *lo = (uint64_t)base;
  *hi = (uint64_t)base + bytes;
  return true;
}


extern "C" {

BSPMM_API const char* bspmm_status_string(bspmm_status_t s) {
  switch (s) {
    case BSPMM_SUCCESS: return "BSPMM_SUCCESS";
    case BSPMM_ERROR_INVALID_VALUE: return "BSPMM_ERROR_INVALID_VALUE";
    case BSPMM_ERROR_OUT_OF_MEMORY: return "BSPMM_ERROR_OUT_OF_MEMORY";
    case BSPMM_ERROR_CUDA: return "BSPMM_ERROR_CUDA";
    case BSPMM_ERROR_INDEX: return "BSPMM_ERROR_INDEX";
    case BSPMM_ERROR_NOT_SUPPORTED: return "BSPMM_ERROR_NOT_SUPPORTED";
  }
  return "BSPMM_UNKNOWN_STATUS";
}

BSPMM_API const char* bspmm_last_error_string(bspmm_handle_t h) { return h ? h->err.c_str() : "null handle"; }

BSPMM_API bspmm_status_t bspmm_create(bspmm_handle_t* out, int device, void* stream, unsigned flags) {
  if (!out) return BSPMM_ERROR_INVALID_VALUE;
  *out = nullptr;
  if (flags & ~BSPMM_VALIDATE) return BSPMM_ERROR_INVALID_VALUE;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return BSPMM_ERROR_NOT_SUPPORTED;
  }
  if (device < 0 || device >= n) return BSPMM_ERROR_INVALID_VALUE;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return BSPMM_ERROR_CUDA;
  if (prop.major != 10 || prop.minor != 0) return BSPMM_ERROR_NOT_SUPPORTED;  // built for sm_100a only
  bspmm_handle_t h = new (std::nothrow) bspmm_handle_s();
  if (!h) return BSPMM_ERROR_OUT_OF_MEMORY;
  h->device = device;
  h->stream = static_cast<cudaStream_t>(stream);
  h->flags = flags;
  h->num_sms = prop.multiProcessorCount;
  h->smem_optin = (int)prop.sharedMemPerBlockOptin;
  DeviceGuard g(device);
  if (cudaMalloc(&h->dev_flag, sizeof(int)) != cudaSuccess ||
      cudaMalloc(&h->dev_sched, sizeof(unsigned long long)) != cudaSuccess) {
    if (h->dev_flag) cudaFree(h->dev_flag);
    delete h;
    return BSPMM_ERROR_OUT_OF_MEMORY;
  }
  cudaMemset(h->dev_flag, 0, sizeof(int));
  cudaMemset(h->dev_sched, 0, sizeof(unsigned long long));
  // the backward's auxiliary stream and fork/join events, created here so that
  // a backward call may be captured into a CUDA graph on its first use
  if (cudaStreamCreateWithFlags(&h->s_aux, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_handoff, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    bspmm_destroy(h);
    return BSPMM_ERROR_CUDA;
  }
  *out = h;
  return BSPMM_SUCCESS;
}

BSPMM_API bspmm_status_t bspmm_destroy(bspmm_handle_t h) {
  if (!h) return BSPMM_SUCCESS;
  bspmm_status_t st = BSPMM_SUCCESS;
  {
    DeviceGuard g(h->device);
    if (cudaStreamSynchronize(h->stream) != cudaSuccess) st = BSPMM_ERROR_CUDA;
    if (h->s_h2d) cudaStreamSynchronize(h->s_h2d), cudaStreamDestroy(h->s_h2d);
    if (h->s_d2h) cudaStreamSynchronize(h->s_d2h), cudaStreamDestroy(h->s_d2h);
    if (h->s_aux) cudaStreamSynchronize(h->s_aux), cudaStreamDestroy(h->s_aux);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    if (h->ev_handoff) cudaEventDestroy(h->ev_handoff);
    for (auto& e : h->ev)
      if (e) cudaEventDestroy(e);
    if (h->ws) cudaFree(h->ws);
    if (h->hbuf) cudaFree(h->hbuf);
    if (h->dev_flag) cudaFree(h->dev_flag);
    if (h->dev_sched) cudaFree(h->dev_sched);
    if (h->scan_ws) cudaFree(h->scan_ws);
    if (h->gcn_ws) cudaFree(h->gcn_ws);
  }
  delete h;
  return st;
}

// The handle's device state (workspace, scan tickets and status words, error
// flag, schedule counter) is shared by its calls, so a call on a new stream must
// not overlap work still queued on the previous one: on a change of stream the
// new stream waits for everything enqueued so far on the old one (one event;
// skipped while either stream is being captured into a CUDA graph, where the
// capture itself orders the work).
BSPMM_API bspmm_status_t bspmm_set_stream(bspmm_handle_t h, void* stream) {
  if (!h) return BSPMM_ERROR_INVALID_VALUE;
  cudaStream_t next = static_cast<cudaStream_t>(stream);
  if (next == h->stream) return BSPMM_SUCCESS;
  DeviceGuard g(h->device);
  cudaStreamCaptureStatus c0 = cudaStreamCaptureStatusNone, c1 = cudaStreamCaptureStatusNone;
  CK(h, cudaStreamIsCapturing(h->stream, &c0));
  CK(h, cudaStreamIsCapturing(next, &c1));
  if (c0 == cudaStreamCaptureStatusNone && c1 == cudaStreamCaptureStatusNone) {
    CK(h, cudaEventRecord(h->ev_handoff, h->stream));
    CK(h, cudaStreamWaitEvent(next, h->ev_handoff, 0));
  }
  h->stream = next;
  return BSPMM_SUCCESS;
}

BSPMM_API bspmm_status_t bspmm_set_hints(bspmm_handle_t h, int32_t max_rows, int64_t max_nnz) {
  if (!h || max_rows < 0 || max_nnz < 0) return BSPMM_ERROR_INVALID_VALUE;
  h->hint_rows = max_rows;
  h->hint_nnz = max_nnz;
  return BSPMM_SUCCESS;
}

BSPMM_API bspmm_status_t bspmm_set_tuning(bspmm_handle_t h, int32_t kt, int32_t warps, int32_t ctas_per_sm,
                                          int32_t chunks) {
  if (!h || kt < 0 || warps < 0 || warps > 16 || ctas_per_sm < 0 || ctas_per_sm > 4 || chunks < 0 || chunks > 4)
    return BSPMM_ERROR_INVALID_VALUE;
  h->tune_kt = kt;
  h->tune_warps = warps;
  h->tune_ctas = ctas_per_sm;
  h->tune_chunks = chunks;
  return BSPMM_SUCCESS;
}

BSPMM_API bspmm_status_t bspmm_set_tile_cb(bspmm_handle_t h, int32_t cb) {
  if (!h || cb < 0 || cb > 32) return BSPMM_ERROR_INVALID_VALUE;
  h->tune_tile_cb = cb;
  return BSPMM_SUCCESS;
}

BSPMM_API bspmm_status_t bspmm_set_trace(bspmm_handle_t h, uint64_t* dev_buf) {
  if (!h) return BSPMM_ERROR_INVALID_VALUE;
  h->trace = reinterpret_cast<unsigned long long*>(dev_buf);
  return BSPMM_SUCCESS;
}

BSPMM_API bspmm_status_t bspmm_set_debug(bspmm_handle_t h, int32_t bits) {
  if (!h || bits < 0 || bits >= (1 << 30)) return BSPMM_ERROR_INVALID_VALUE;
  h->dbg = bits;
  return BSPMM_SUCCESS;
}

BSPMM_API bspmm_status_t bspmm_set_gcn_math(bspmm_handle_t h, int32_t mode) {
  if (!h || mode < BSPMM_GCN_FP32 || mode > BSPMM_GCN_BF16) return BSPMM_ERROR_INVALID_VALUE;
  h->gcn_math = mode;
  return BSPMM_SUCCESS;
}

BSPMM_API bspmm_status_t bspmm_sync(bspmm_handle_t h) {
  if (!h) return BSPMM_ERROR_INVALID_VALUE;
  DeviceGuard g(h->device);
  CK(h, sync_streams(h));
  CK(h, cudaGetLastError());
  if (h->coo_fused_pending) {  // a fused bspmm_coo skipped a matrix beyond the planner hints?
    h->coo_fused_pending = false;
    int flag = 0;
    CK(h, cudaMemcpy(&flag, h->dev_flag, sizeof(int), cudaMemcpyDeviceToHost));
    if (flag & 64) {
      CK(h, cudaMemset(h->dev_flag, 0, sizeof(int)));
      return fail(h, BSPMM_ERROR_INVALID_VALUE,
                  "bspmm_coo: a matrix exceeded the max_rows / max_nnz hints; its rows were not written");
    }
  }
  return BSPMM_SUCCESS;
}

BSPMM_API bspmm_status_t bspmm_last_plan(bspmm_handle_t h, bspmm_plan_t* out) {
  if (!h || !out) return BSPMM_ERROR_INVALID_VALUE;
  *out = h->last_plan;
  return BSPMM_SUCCESS;
}

BSPMM_API int64_t bspmm_launch_count(bspmm_handle_t h) { return h ? h->launches : -1; }

BSPMM_API bspmm_status_t bspmm_build_offsets(bspmm_handle_t h, int32_t batch, const int32_t* sizes,
                                             int64_t* offsets_out) {
  if (!h || batch < 0 || !offsets_out || (batch > 0 && !sizes)) return BSPMM_ERROR_INVALID_VALUE;
  DeviceGuard g(h->device);
  if ((h->flags & BSPMM_VALIDATE) && batch > 0) {
    CK(h, cudaMemsetAsync(h->dev_flag, 0, sizeof(int), h->stream));
    CK(h, launch_validate_sizes(batch, sizes, h->dev_flag, h->stream));
    h->launches++;
    bspmm_status_t st = check_validate_flag(h);
    if (st != BSPMM_SUCCESS) return st;
  }
  if (batch == 0) {
    CK(h, cudaMemsetAsync(offsets_out, 0, sizeof(int64_t), h->stream));
    return BSPMM_SUCCESS;
  }
  ScanState ss;
  bspmm_status_t st = scan_state(h, batch, &ss);
  if (st != BSPMM_SUCCESS) return st;
  CK(h, launch_offsets(batch, sizes, offsets_out, ss, h->stream));
  h->launches++;
  return BSPMM_SUCCESS;
}

static bspmm_status_t csr_impl(bspmm_handle_t h, int32_t batch, int32_t k, const int64_t* row_off,
                               const int32_t* sizes, const int32_t* row_ptr, const int32_t* col_idx,
                               const float* vals, const float* B, int64_t ldb, float* C, int64_t ldc,
                               bool validate, const float* bias = nullptr, int32_t accumulate = 0,
                               int32_t mc = 0) {
  if (validate) {
    CK(h, cudaMemsetAsync(h->dev_flag, 0, sizeof(int), h->stream));
    CK(h, launch_validate_csr(batch, row_off, sizes, row_ptr, col_idx, h->dev_flag, h->stream));
    h->launches++;
    bspmm_status_t st = check_validate_flag(h);
    if (st != BSPMM_SUCCESS) return st;
  }
  const bool aligned = (k % 4 == 0) && (ldb % 4 == 0) && (ldc % 4 == 0) && aligned16(B) && aligned16(C);
  bspmm_plan_t plan;
  bspmm_status_t st = plan_for(h, batch, k, aligned, &plan);
  if (st != BSPMM_SUCCESS) return st;
  // small batches (every tile resident at once): the tile kernel
  // (spmm_tile.cu); tuning overrides and the debug bits of the pipeline kernel
  // keep the pipeline
  TileLayout L;
  const bool tuned = h->tune_kt || h->tune_warps || h->tune_ctas || h->tune_chunks;
  if (plan.vec && mc == 0 && !tuned && !(h->dbg & (2 | 4 | 8 | 128 | 16384)) &&
      plan_tile(batch, k, h->hint_rows, h->hint_nnz, h->num_sms, h->tune_tile_cb, &L)) {
    plan.kernel = 1;
    plan.kt = 4 * L.cb;
    plan.tiles = L.tiles;
    plan.lanes = L.cb;
    plan.chunks = 1;
    plan.stages = 1;
    plan.units = L.units;
    plan.grid = (int32_t)L.units;
    plan.threads = 128;
    plan.smem_bytes = L.smem;
    h->last_plan = plan;
    const TmaMaps* maps = (L.cb >= 8 && !(h->dbg & 32768)) ? tma_maps(h, B, k, ldb, 4 * L.cb) : nullptr;
    CsrArgs a{batch, k, row_off, sizes, row_ptr, col_idx, vals, B, ldb, C, ldc, h->trace, h->dbg, maps, bias,
              accumulate};
    if (prewait_prefetch(h)) {
      alloc_range(h, B, &a.b_lo, &a.b_hi);
      if (!(h->dbg & kDbgNoStructPrefetch) && alloc_range(h, row_ptr, &a.s_lo[0], &a.s_hi[0])) {
        alloc_range(h, col_idx, &a.s_lo[1], &a.s_hi[1]);
        alloc_range(h, vals, &a.s_lo[2], &a.s_hi[2]);
      }
    }
    CK(h, launch_spmm_tile(a, L, h->stream));
    h->launches++;
    return BSPMM_SUCCESS;
  }
  const TmaMaps* maps = plan.vec ? tma_maps(h, B, k, ldb, plan.kt) : nullptr;
  if (h->dbg & 64) plan.sched = 0;
  if ((h->dbg & 128) && row_off) plan.sched = 1;
  h->last_plan = plan;
  CsrArgs a{batch, k, row_off, sizes, row_ptr, col_idx, vals, B, ldb, C, ldc, h->trace, h->dbg, maps, bias, accumulate,
            plan.sched ? h->dev_sched : nullptr};
  a.mc = mc;
  if (prewait_prefetch(h)) {
    alloc_range(h, B, &a.b_lo, &a.b_hi);
    if (!(h->dbg & kDbgNoStructPrefetch)) alloc_range(h, row_ptr, &a.s_lo[0], &a.s_hi[0]);
  }
  CK(h, launch_spmm_csr(a, plan, h->stream));
  if (plan.units > 0) h->launches++;
  return BSPMM_SUCCESS;
}

static bspmm_status_t csr_entry(bspmm_handle_t h, int32_t batch, int32_t k, const int64_t* row_off,
                                const int32_t* sizes, const int32_t* row_ptr, const int32_t* col_idx,
                                const float* vals, const float* B, int64_t ldb, float* C, int64_t ldc, int32_t mc) {
  if (!h) return BSPMM_ERROR_INVALID_VALUE;
  if (batch < 0 || k < 1 || ldb < k || ldc < k) return fail(h, BSPMM_ERROR_INVALID_VALUE, "batch<0, k<1 or ld<k");
  if (batch == 0) return BSPMM_SUCCESS;
  // col_idx / vals / B / C may be NULL only when they have no elements (caller's promise)
  if ((!row_off && !sizes) || !row_ptr) return fail(h, BSPMM_ERROR_INVALID_VALUE, "NULL pointer argument");
  if (B && B == C) return fail(h, BSPMM_ERROR_INVALID_VALUE, "C must not alias B");
  DeviceGuard g(h->device);
  if (!row_off && (h->flags & BSPMM_VALIDATE)) {  // validation needs materialised offsets
    bspmm_status_t st = grow(h, &h->ws, &h->ws_bytes, al256((size_t)(batch + 1) * 8));
    if (st != BSPMM_SUCCESS) return st;
    int64_t* ro = static_cast<int64_t*>(h->ws);
    st = bspmm_build_offsets(h, batch, sizes, ro);
    if (st != BSPMM_SUCCESS) return st;
    return csr_impl(h, batch, k, ro, nullptr, row_ptr, col_idx, vals, B, ldb, C, ldc, true, nullptr, 0, mc);
  }
  if (!row_off) {
    // row_off == NULL: small batches (every CTA's units fit one metadata batch)
    // build the packed offsets inside the SpMM producer (fused row a-1, one
    // launch); large ones use the look-back scan kernel first -- the fused
    // prefix costs dependent round trips on the producer's path every 32 units
    // (C5: 866 vs 832 us per step, tools/kbench.py)
    const bool aligned = (k % 4 == 0) && (ldb % 4 == 0) && (ldc % 4 == 0) && aligned16(B) && aligned16(C);
    bspmm_plan_t pl;
    bspmm_status_t st = make_plan(k, batch, aligned, h->hint_rows, h->hint_nnz, h->num_sms, h->smem_optin,
                                  h->tune_kt, h->tune_warps, h->tune_ctas, h->tune_chunks, &pl);
    if (st != BSPMM_SUCCESS) return fail(h, st, "planner rejected the arguments");
    if (pl.units > 32LL * pl.grid) {
      st = grow(h, &h->ws, &h->ws_bytes, al256((size_t)(batch + 1) * 8));
      if (st != BSPMM_SUCCESS) return st;
      int64_t* ro = static_cast<int64_t*>(h->ws);
      st = bspmm_build_offsets(h, batch, sizes, ro);
      if (st != BSPMM_SUCCESS) return st;
      return csr_impl(h, batch, k, ro, nullptr, row_ptr, col_idx, vals, B, ldb, C, ldc, false, nullptr, 0, mc);
    }
  }
  return csr_impl(h, batch, k, row_off, sizes, row_ptr, col_idx, vals, B, ldb, C, ldc,
                  (h->flags & BSPMM_VALIDATE) != 0, nullptr, 0, mc);
}

BSPMM_API bspmm_status_t bspmm_csr(bspmm_handle_t h, int32_t batch, int32_t k, const int64_t* row_off,
                                   const int32_t* sizes, const int32_t* row_ptr, const int32_t* col_idx,
                                   const float* vals, const float* B, int64_t ldb, float* C, int64_t ldc) {
  return csr_entry(h, batch, k, row_off, sizes, row_ptr, col_idx, vals, B, ldb, C, ldc, 0);
}

BSPMM_API bspmm_status_t bspmm_csr_multicast(bspmm_handle_t h, int32_t batch, int32_t k, const int64_t* row_off,
                                             const int32_t* sizes, const int32_t* row_ptr, const int32_t* col_idx,
                                             const float* vals, const float* B, int64_t ldb, float* C_mc,
                                             int64_t ldc) {
  return csr_entry(h, batch, k, row_off, sizes, row_ptr, col_idx, vals, B, ldb, C_mc, ldc, 1);
}

// workspace layout for the COO path: [row_off][row_ptr][col][val][keys x2][pay x2]
struct CooWs {
  int64_t* row_off;
  int32_t* row_ptr;
  int32_t* col;
  float* val;
  uint64_t* keys;
  uint32_t* pay;
};

static bspmm_status_t coo_workspace(bspmm_handle_t h, int32_t batch, int64_t N, int64_t NNZ, bool need_ro,
                                    bool need_csr, CooWs* w) {
  size_t off = 0;
  const size_t o_ro = off;
  off += need_ro ? al256((size_t)(batch + 1) * 8) : 0;
  const size_t o_rp = off;
  off += need_csr ? al256((size_t)(N + 1) * 4) : 0;
  const size_t o_col = off;
  off += need_csr ? al256((size_t)NNZ * 4) : 0;
  const size_t o_val = off;
  off += need_csr ? al256((size_t)NNZ * 4) : 0;
  const size_t o_keys = off;
  off += al256((size_t)2 * NNZ * 8);
  const size_t o_pay = off;
  off += al256((size_t)2 * NNZ * 4);
  bspmm_status_t st = grow(h, &h->ws, &h->ws_bytes, std::max<size_t>(off, 256));
  if (st != BSPMM_SUCCESS) return st;
  char* b = static_cast<char*>(h->ws);
  w->row_off = need_ro ? reinterpret_cast<int64_t*>(b + o_ro) : nullptr;
  w->row_ptr = need_csr ? reinterpret_cast<int32_t*>(b + o_rp) : nullptr;
  w->col = need_csr ? reinterpret_cast<int32_t*>(b + o_col) : nullptr;
  w->val = need_csr ? reinterpret_cast<float*>(b + o_val) : nullptr;
  w->keys = reinterpret_cast<uint64_t*>(b + o_keys);
  w->pay = reinterpret_cast<uint32_t*>(b + o_pay);
  return BSPMM_SUCCESS;
}

static bspmm_status_t coo2csr_impl(bspmm_handle_t h, int32_t batch, const int64_t* row_off, const int32_t* sizes,
                                   const int64_t* nnz_off, const int32_t* idx, const float* vals, int64_t NNZ,
                                   int32_t* rp, int32_t* col, float* val, const CooWs& w) {
  if (h->flags & BSPMM_VALIDATE) {
    CK(h, cudaMemsetAsync(h->dev_flag, 0, sizeof(int), h->stream));
    CK(h, launch_validate_coo(batch, row_off, sizes, nnz_off, idx, h->dev_flag, h->stream));
    h->launches++;
    bspmm_status_t st = check_validate_flag(h);
    if (st != BSPMM_SUCCESS) return st;
  }
  const int32_t cap = coo_smem_cap(h->hint_nnz, h->smem_optin);
  CK(h, launch_coo2csr(batch, row_off, sizes, nnz_off, idx, vals, rp, col, val, w.keys, w.pay, NNZ, cap,
                       h->stream));
  h->launches++;
  return BSPMM_SUCCESS;
}

BSPMM_API bspmm_status_t bspmm_coo2csr(bspmm_handle_t h, int32_t batch, const int64_t* row_off,
                                       const int32_t* sizes, const int64_t* nnz_off, const int32_t* idx,
                                       const float* vals, int64_t total_rows, int64_t total_nnz,
                                       int32_t* row_ptr_out, int32_t* col_out, float* val_out) {
  if (!h) return BSPMM_ERROR_INVALID_VALUE;
  if (batch < 0 || total_rows < 0 || total_nnz < 0 || total_nnz > INT32_MAX)
    return fail(h, BSPMM_ERROR_INVALID_VALUE, "bad batch / totals");
  if (batch == 0) return BSPMM_SUCCESS;
  if (!row_off || !nnz_off || !row_ptr_out || (total_nnz > 0 && (!idx || !vals || !col_out || !val_out)))
    return fail(h, BSPMM_ERROR_INVALID_VALUE, "NULL pointer argument");
  DeviceGuard g(h->device);
  CooWs w;
  bspmm_status_t st = coo_workspace(h, batch, total_rows, total_nnz, false, false, &w);
  if (st != BSPMM_SUCCESS) return st;
  return coo2csr_impl(h, batch, row_off, sizes, nnz_off, idx, vals, total_nnz, row_ptr_out, col_out, val_out, w);
}

BSPMM_API bspmm_status_t bspmm_coo(bspmm_handle_t h, int32_t batch, int32_t k, const int64_t* row_off,
                                   const int32_t* sizes, const int64_t* nnz_off, const int32_t* idx,
                                   const float* vals, const float* B, int64_t ldb, float* C, int64_t ldc,
                                   int64_t total_rows, int64_t total_nnz, int32_t* csr_row_ptr_out,
                                   int32_t* csr_col_out, float* csr_val_out) {
  if (!h) return BSPMM_ERROR_INVALID_VALUE;
  if (batch < 0 || k < 1 || ldb < k || ldc < k || total_rows < 0 || total_nnz < 0 || total_nnz > INT32_MAX)
    return fail(h, BSPMM_ERROR_INVALID_VALUE, "batch<0, k<1, ld<k or bad totals");
  if (batch == 0) return BSPMM_SUCCESS;
  const bool out_given = csr_row_ptr_out != nullptr;
  if (out_given != (csr_col_out != nullptr) || out_given != (csr_val_out != nullptr))
    return fail(h, BSPMM_ERROR_INVALID_VALUE, "csr_*_out must be all NULL or all non-NULL");
  if ((!row_off && !sizes) || !nnz_off || !B || !C || (total_nnz > 0 && (!idx || !vals)))
    return fail(h, BSPMM_ERROR_INVALID_VALUE, "NULL pointer argument");
  if (B && B == C) return fail(h, BSPMM_ERROR_INVALID_VALUE, "C must not alias B");
  DeviceGuard g(h->device);
  CooWs w;
  bspmm_status_t st = coo_workspace(h, batch, total_rows, total_nnz, row_off == nullptr, !out_given, &w);
  if (st != BSPMM_SUCCESS) return st;
  const int64_t* ro = row_off;
  if (!ro) {
    st = bspmm_build_offsets(h, batch, sizes, w.row_off);
    if (st != BSPMM_SUCCESS) return st;
    ro = w.row_off;
  }
  // Fused path (one SpMM launch converts each matrix's SparseTensor slice to CSR
  // in shared memory): needs the vectorised path, planner hints that bound every
  // matrix (a matrix beyond them is skipped and reported by bspmm_sync), and no
  // request for the built CSR.
  const bool aligned = (k % 4 == 0) && (ldb % 4 == 0) && (ldc % 4 == 0) && aligned16(B) && aligned16(C);
  if (!out_given && aligned && h->hint_rows > 0 && h->hint_nnz > 0 && !(h->flags & BSPMM_VALIDATE)) {
    // small batches (every tile resident at once): the tile kernel's SparseTensor
    // variant (spmm_tile.cu, each tile CTA converts its matrix while its B tile
    // lands); debug bit 16384 keeps the pipeline's converter warps
    TileLayout TL;
    const bool tuned = h->tune_kt || h->tune_warps || h->tune_ctas || h->tune_chunks;
    if (!tuned && !(h->dbg & (16384 | 128)) &&
        plan_tile(batch, k, h->hint_rows, h->hint_nnz, h->num_sms, h->tune_tile_cb, &TL, /*coo=*/true)) {
      bspmm_plan_t plan{};
      plan.kernel = 1;
      plan.kt = 4 * TL.cb;
      plan.tiles = TL.tiles;
      plan.lanes = TL.cb;
      plan.vec = 1;
      plan.chunks = 1;
      plan.stages = 1;
      plan.units = TL.units;
      plan.grid = (int32_t)TL.units;
      plan.threads = 128;
      plan.smem_bytes = TL.smem;
      plan.max_rows = h->hint_rows;
      h->last_plan = plan;
      const TmaMaps* maps = (TL.cb >= 8 && !(h->dbg & 32768)) ? tma_maps(h, B, k, ldb, 4 * TL.cb) : nullptr;
      CsrArgs a{batch, k, ro, sizes, nullptr, nullptr, vals, B, ldb, C, ldc, h->trace, h->dbg, maps};
      a.coo_nnz_off = nnz_off;
      a.coo_idx = idx;
      a.err = h->dev_flag;
      if (prewait_prefetch(h)) {
        alloc_range(h, B, &a.b_lo, &a.b_hi);
        if (!(h->dbg & kDbgNoStructPrefetch) && alloc_range(h, idx, &a.s_lo[1], &a.s_hi[1]))
          alloc_range(h, vals, &a.s_lo[2], &a.s_hi[2]);
      }
      CK(h, launch_spmm_tile(a, TL, h->stream));
      h->launches++;
      h->coo_fused_pending = true;
      return BSPMM_SUCCESS;
    }
    bspmm_plan_t plan;
    st = make_plan(k, batch, true, h->hint_rows, h->hint_nnz, h->num_sms, h->smem_optin, h->tune_kt, h->tune_warps,
                   h->tune_ctas, h->tune_chunks, &plan, /*coo=*/true);
    if (st != BSPMM_SUCCESS) return fail(h, st, "planner rejected the arguments");
    if ((int64_t)plan.stage_b_bytes >= (int64_t)h->hint_rows * plan.kt * 4) {
      h->last_plan = plan;
      const TmaMaps* maps = tma_maps(h, B, k, ldb, plan.kt);
      CsrArgs a{batch, k, ro, sizes, nullptr, nullptr, vals, B, ldb, C, ldc, h->trace, h->dbg, maps};
      a.coo_nnz_off = nnz_off;
      a.coo_idx = idx;
      a.err = h->dev_flag;
      a.cvt_warps = kCooWarps - 1 - coo_consumer_warps(h->tune_warps);
      if (h->dbg & 128) {  // dynamic unit schedule (global ticket counter)
        plan.sched = 1;
        h->last_plan = plan;
        a.sched = h->dev_sched;
      }
      if (prewait_prefetch(h)) {
        alloc_range(h, B, &a.b_lo, &a.b_hi);
        if (!(h->dbg & kDbgNoStructPrefetch) && alloc_range(h, idx, &a.s_lo[1], &a.s_hi[1]))
          alloc_range(h, vals, &a.s_lo[2], &a.s_hi[2]);
      }
      CK(h, launch_spmm_csr(a, plan, h->stream));
      if (plan.units > 0) h->launches++;
      h->coo_fused_pending = true;
      return BSPMM_SUCCESS;
    }
  }
  int32_t* rp = out_given ? csr_row_ptr_out : w.row_ptr;
  int32_t* col = out_given ? csr_col_out : w.col;
  float* val = out_given ? csr_val_out : w.val;
  st = coo2csr_impl(h, batch, ro, sizes, nnz_off, idx, vals, total_nnz, rp, col, val, w);
  if (st != BSPMM_SUCCESS) return st;
  // indices were validated on the COO side; the built CSR is consistent by construction
  return csr_impl(h, batch, k, ro, sizes, rp, col, val, B, ldb, C, ldc, false);
}

// ---- fused batched GCN layer (NEXT-1) ----------------------------------------
// PAPER.md Fig. algo:graph_conv_batched: for ch: U = X W[ch]; B = U + bias[ch];
// C[ch] = BatchedSpMM(A[ch], B); Y = sum_ch C[ch].  Here (gcn_fused.cu): one
// preparation launch (W to K-major + TF32 split, tile table) and ONE fused
// tcgen05 launch computing Y = [A_ch X | rowsum(A_ch)] . [W_ch; bias_ch] per
// 128-row x nt-feature tile, Z produced by the SpMM row loop straight into the
// tensor core's shared-memory operand, the channel sum and bias in the TMEM
// accumulation.  No library GEMM, no U round trip through HBM.
BSPMM_API bspmm_status_t bspmm_gcn_layer(bspmm_handle_t h, int32_t batch, int32_t channels, int32_t n_x, int32_t k,
                                         const int64_t* row_off, const int32_t* sizes, const int32_t* row_ptr,
                                         const int32_t* col, const float* vals, const float* X, int64_t ldx,
                                         const float* W, const float* bias, float* Y, int64_t ldy,
                                         int64_t total_rows) {
  if (!h) return BSPMM_ERROR_INVALID_VALUE;
  if (batch < 0 || channels < 1 || n_x < 1 || k < 1 || ldx < n_x || ldy < k || total_rows < 0)
    return fail(h, BSPMM_ERROR_INVALID_VALUE, "bad batch / channels / sizes / leading dimensions");
  if (batch == 0 || total_rows == 0) return BSPMM_SUCCESS;
  if (!row_off || !row_ptr || !X || !W || !Y) return fail(h, BSPMM_ERROR_INVALID_VALUE, "NULL pointer argument");
  if (total_rows >= INT32_MAX) return fail(h, BSPMM_ERROR_NOT_SUPPORTED, "bspmm_gcn_layer: total_rows >= 2^31");
  DeviceGuard g(h->device);
  const int64_t N = total_rows;
  if (h->flags & BSPMM_VALIDATE) {
    for (int32_t ch = 0; ch < channels; ++ch) {
      CK(h, cudaMemsetAsync(h->dev_flag, 0, sizeof(int), h->stream));
      CK(h, launch_validate_csr(batch, row_off, sizes, row_ptr + (int64_t)ch * (N + 1), col, h->dev_flag, h->stream));
      h->launches++;
      bspmm_status_t st = check_validate_flag(h);
      if (st != BSPMM_SUCCESS) return st;
    }
  }
  GcnPlan L;
  // debug bits 20-21: feature-tile width override (1: 64, 2: 128, 3: 256)
  const int32_t nt_ovr = ((h->dbg >> 20) & 3) ? (32 << ((h->dbg >> 20) & 3)) : 0;
  // CTA pairs (tcgen05 cta_group::2, M = 256, each CTA staging half of W) for
  // the fp32 (3xTF32) layer over many row tiles: 65536 graphs 27.0-27.1 vs
  // 27.4-28.2 ms; the one-pass modes and small batches measured slower with
  // pairs (TF32 20.8 vs 17.3 ms; Reaction100-like 92.8 vs 70.7 us), so they
  // keep one CTA per tile.  Debug bit 1<<22 forces pairs, 1<<23 single CTAs.
  const bool big = (N + 127) / 128 >= 4LL * h->num_sms;
  int32_t cg = (h->gcn_math == BSPMM_GCN_FP32 && big) ? 2 : 1;
  if (h->dbg & (1 << 22)) cg = 2;
  if (h->dbg & (1 << 23)) cg = 1;
  if (!plan_gcn(channels, n_x, k, N, h->hint_rows, h->smem_optin, h->gcn_math, h->num_sms, nt_ovr, cg, &L))
    return fail(h, BSPMM_ERROR_NOT_SUPPORTED, "bspmm_gcn_layer: no shared-memory plan for these sizes");
  // X needs a 16-byte row pitch and base for TMA; otherwise a packed copy
  const bool x_ok = (ldx % 4 == 0) && aligned16(X);
  const int64_t ldxp = x_ok ? ldx : (n_x + 3) / 4 * 4;
  // workspace: [Wt_hi k x ktot][Wt_lo k x ktot (3xTF32)][gfirst tiles_m][packed X]
  const size_t wt_bytes = al256((size_t)k * L.ktot * 4);
  const size_t o_hi = 0, o_lo = wt_bytes, o_gf = o_lo + (h->gcn_math == BSPMM_GCN_FP32 ? wt_bytes : 0);
  const size_t o_x = o_gf + al256((size_t)L.tiles_m * 4);
  const size_t bytes = o_x + (x_ok ? 0 : al256((size_t)N * ldxp * 4));
  bspmm_status_t st = grow(h, &h->gcn_ws, &h->gcn_ws_bytes, bytes);
  if (st != BSPMM_SUCCESS) return st;
  char* wsb = static_cast<char*>(h->gcn_ws);
  float* whi = reinterpret_cast<float*>(wsb + o_hi);
  float* wlo = h->gcn_math == BSPMM_GCN_FP32 ? reinterpret_cast<float*>(wsb + o_lo) : whi;
  int32_t* gfirst = reinterpret_cast<int32_t*>(wsb + o_gf);
  const float* Xk = x_ok ? X : reinterpret_cast<const float*>(wsb + o_x);
  CUtensorMap mx, mhi, mlo;
  if (!encode_2d(&mx, Xk, (uint64_t)n_x, (uint64_t)N, (uint64_t)ldxp * 4, 32, 64, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_2d(&mhi, whi, (uint64_t)L.ktot, (uint64_t)k, (uint64_t)L.ktot * 4, 32, (uint32_t)(L.nt / L.cg),
                 CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_2d(&mlo, wlo, (uint64_t)L.ktot, (uint64_t)k, (uint64_t)L.ktot * 4, 32, (uint32_t)(L.nt / L.cg),
                 CU_TENSOR_MAP_SWIZZLE_128B))
    return fail(h, BSPMM_ERROR_CUDA, "bspmm_gcn_layer: TMA descriptor encoding failed");
  if (!x_ok) {
    CK(h, launch_gcn_pack_x(X, ldx, n_x, N, const_cast<float*>(Xk), ldxp, h->num_sms, h->stream));
    h->launches++;
  }
  CK(h, launch_gcn_prep(L, batch, channels, n_x, k, N, h->gcn_math, W, bias, whi, wlo, row_off, gfirst, h->stream));
  h->launches++;
  GcnArgs a{batch, channels, n_x, k, h->gcn_math, (h->dbg >> 17) & 7, N, row_off, sizes, row_ptr, col, vals, Xk, ldxp, Y, ldy, gfirst,
            &mx, &mhi, &mlo};
  CK(h, launch_gcn_fused(L, a, h->stream));
  h->launches++;
  return BSPMM_SUCCESS;
}

// ---- the paper's atomic SWA SpMM for SparseTensor (NEXT-3) -----------------
BSPMM_API bspmm_status_t bspmm_coo_atomic(bspmm_handle_t h, int32_t batch, int32_t k, const int64_t* row_off,
                                          const int32_t* sizes, const int64_t* nnz_off, const int32_t* idx,
                                          const float* vals, const float* B, int64_t ldb, float* C, int64_t ldc) {
  if (!h) return BSPMM_ERROR_INVALID_VALUE;
  if (batch < 0 || k < 1 || ldb < k || ldc < k) return fail(h, BSPMM_ERROR_INVALID_VALUE, "batch<0, k<1 or ld<k");
  if (batch == 0) return BSPMM_SUCCESS;
  if ((!row_off && !sizes) || !nnz_off) return fail(h, BSPMM_ERROR_INVALID_VALUE, "NULL pointer argument");
  if (B && B == C) return fail(h, BSPMM_ERROR_INVALID_VALUE, "C must not alias B");
  if (!(k % 4 == 0 && ldb % 4 == 0 && ldc % 4 == 0 && aligned16(B) && aligned16(C)))
    return fail(h, BSPMM_ERROR_NOT_SUPPORTED, "bspmm_coo_atomic needs k, ldb, ldc % 4 == 0 and 16-byte aligned B, C");
  DeviceGuard g(h->device);
  const int64_t* ro = row_off;
  if (!ro) {
    bspmm_status_t st = grow(h, &h->ws, &h->ws_bytes, al256((size_t)(batch + 1) * 8));
    if (st != BSPMM_SUCCESS) return st;
    int64_t* w = static_cast<int64_t*>(h->ws);
    st = bspmm_build_offsets(h, batch, sizes, w);
    if (st != BSPMM_SUCCESS) return st;
    ro = w;
  }
  if (h->flags & BSPMM_VALIDATE) {
    CK(h, cudaMemsetAsync(h->dev_flag, 0, sizeof(int), h->stream));
    CK(h, launch_validate_coo(batch, ro, sizes, nnz_off, idx, h->dev_flag, h->stream));
    h->launches++;
    bspmm_status_t st = check_validate_flag(h);
    if (st != BSPMM_SUCCESS) return st;
  }
  CK(h, launch_spmm_coo_atomic(batch, k, ro, sizes, nnz_off, idx, vals, B, ldb, C, ldc, h->hint_rows, h->smem_optin,
                               h->stream));
  h->launches++;
  return BSPMM_SUCCESS;
}

// ---- backward (NEXT-2) ------------------------------------------------------
// workspace (grad_B only): rowT (N+1) i32, colT NNZ i32, valsT NNZ f32 -- the internal A^T
struct TransWs {
  int32_t *rowT, *colT;
  float* valsT;
};

static bspmm_status_t trans_workspace(bspmm_handle_t h, int64_t N, int64_t NNZ, TransWs* w) {
  size_t off = 0;
  const size_t o_rt = off;
  off += al256((size_t)(N + 1) * 4);
  const size_t o_ct = off;
  off += al256((size_t)NNZ * 4 + 4);
  const size_t o_vt = off;
  off += al256((size_t)NNZ * 4 + 4);
  bspmm_status_t st = grow(h, &h->ws, &h->ws_bytes, off);
  if (st != BSPMM_SUCCESS) return st;
  char* b = static_cast<char*>(h->ws);
  w->rowT = reinterpret_cast<int32_t*>(b + o_rt);
  w->colT = reinterpret_cast<int32_t*>(b + o_ct);
  w->valsT = reinterpret_cast<float*>(b + o_vt);
  return BSPMM_SUCCESS;
}

static bspmm_status_t transpose_impl(bspmm_handle_t h, int32_t batch, const int64_t* row_off, const int32_t* sizes,
                                     const int32_t* row_ptr, const int32_t* col, const float* vals, int32_t* rowT,
                                     int32_t* colT, float* valsT, cudaStream_t stream = nullptr) {
  if (!stream) stream = h->stream;
  if (h->flags & BSPMM_VALIDATE) {
    CK(h, cudaMemsetAsync(h->dev_flag, 0, sizeof(int), h->stream));
    CK(h, launch_validate_csr(batch, row_off, sizes, row_ptr, col, h->dev_flag, h->stream));
    h->launches++;
    bspmm_status_t st = check_validate_flag(h);
    if (st != BSPMM_SUCCESS) return st;
  }
  CK(h, launch_transpose_csr(batch, row_off, sizes, row_ptr, col, vals, rowT, colT, valsT, h->hint_rows, h->hint_nnz,
                             h->num_sms, stream));
  h->launches++;
  return BSPMM_SUCCESS;
}

BSPMM_API bspmm_status_t bspmm_csr_transpose(bspmm_handle_t h, int32_t batch, const int64_t* row_off,
                                             const int32_t* sizes, const int32_t* row_ptr, const int32_t* col,
                                             const float* vals, int64_t total_rows, int64_t total_nnz,
                                             int32_t* rowT_out, int32_t* colT_out, float* valsT_out) {
  if (!h) return BSPMM_ERROR_INVALID_VALUE;
  if (batch < 0 || total_rows < 0 || total_nnz < 0 || total_nnz > INT32_MAX)
    return fail(h, BSPMM_ERROR_INVALID_VALUE, "bad batch / totals");
  if (batch == 0) return BSPMM_SUCCESS;
  if (!row_off || !row_ptr || !rowT_out || (total_nnz > 0 && (!col || !vals || !colT_out || !valsT_out)))
    return fail(h, BSPMM_ERROR_INVALID_VALUE, "NULL pointer argument");
  DeviceGuard g(h->device);
  return transpose_impl(h, batch, row_off, sizes, row_ptr, col, vals, rowT_out, colT_out, valsT_out);
}

BSPMM_API bspmm_status_t bspmm_sddmm(bspmm_handle_t h, int32_t batch, int32_t k, const int64_t* row_off,
                                     const int32_t* sizes, const int32_t* row_ptr, const int32_t* col, const float* B,
                                     int64_t ldb, const float* G, int64_t ldg, float* out) {
  if (!h) return BSPMM_ERROR_INVALID_VALUE;
  if (batch < 0 || k < 1 || ldb < k || ldg < k) return fail(h, BSPMM_ERROR_INVALID_VALUE, "batch<0, k<1 or ld<k");
  if (batch == 0) return BSPMM_SUCCESS;
  if (!row_off || !row_ptr) return fail(h, BSPMM_ERROR_INVALID_VALUE, "NULL pointer argument");
  DeviceGuard g(h->device);
  if (h->flags & BSPMM_VALIDATE) {
    CK(h, cudaMemsetAsync(h->dev_flag, 0, sizeof(int), h->stream));
    CK(h, launch_validate_csr(batch, row_off, sizes, row_ptr, col, h->dev_flag, h->stream));
    h->launches++;
    bspmm_status_t st = check_validate_flag(h);
    if (st != BSPMM_SUCCESS) return st;
  }
  if (!out) return BSPMM_SUCCESS;  // no entries (caller's promise)
  // latency-bound batches (<= 8 matrices per SM): whole-row units of the SpMM
  // pipeline (TMA-staged B_i in the ring, the consumers' SDDMM mode; C2 8.8
  // -> 5.6 us, C3 63.6 -> 19 us, C4 12.4 -> 10.5 us).  Streaming batches, k >
  // 512, unaligned or split plans: the standalone kernel below (C5: 1071 vs
  // 1650 us; also forced by debug bit 256)
  const bool aligned = (k % 4 == 0) && (ldb % 4 == 0) && (ldg % 4 == 0) && aligned16(B) && aligned16(G);
  if (aligned && k <= kMaxVecKt && (batch <= 8 * h->num_sms || (h->dbg & 1024)) && !(h->dbg & 256)) {
    bspmm_plan_t plan;
    bspmm_status_t st = make_plan(k, batch, true, h->hint_rows, h->hint_nnz, h->num_sms, h->smem_optin, k,
                                  h->tune_warps, h->tune_ctas, h->tune_chunks, &plan);
    if (st == BSPMM_SUCCESS && plan.vec && plan.tiles == 1) {
      const TmaMaps* maps = tma_maps(h, B, k, ldb, plan.kt);
      // the staged CSR slice carries a values array: point it at col (read, never used)
      CsrArgs a{batch, k, row_off, sizes, row_ptr, col, reinterpret_cast<const float*>(col), B, ldb, nullptr, k,
                h->trace, h->dbg, maps};
      a.G = G;
      a.ldg = ldg;
      a.sd_out = out;
      if (prewait_prefetch(h) && alloc_range(h, B, &a.b_lo, &a.b_hi)) {
        alloc_range(h, G, &a.g_lo, &a.g_hi);
        if (!(h->dbg & kDbgNoStructPrefetch)) alloc_range(h, row_ptr, &a.s_lo[0], &a.s_hi[0]);
      }
      h->last_plan = plan;
      CK(h, launch_spmm_csr(a, plan, h->stream));
      if (plan.units > 0) h->launches++;
      return BSPMM_SUCCESS;
    }
  }
  CK(h, launch_sddmm(batch, k, row_off, sizes, row_ptr, col, B, ldb, G, ldg, out, h->hint_rows, h->hint_nnz,
                     h->num_sms, h->dbg,
                     h->stream));
  h->launches++;
  return BSPMM_SUCCESS;
}

// grad_B = A^T grad_C by the forward kernel, without the pre-wait prefetch
static bspmm_status_t csr_impl_bwd(bspmm_handle_t h, int32_t batch, int32_t k, const int64_t* row_off,
                                   const int32_t* sizes, const int32_t* rowT, const int32_t* colT, const float* valsT,
                                   const float* G, int64_t ldg, float* gB, int64_t ldgb) {
  h->in_backward = true;
  const bspmm_status_t st = csr_impl(h, batch, k, row_off, sizes, rowT, colT, valsT, G, ldg, gB, ldgb, false);
  h->in_backward = false;
  return st;
}

BSPMM_API bspmm_status_t bspmm_csr_backward(bspmm_handle_t h, int32_t batch, int32_t k, const int64_t* row_off,
                                            const int32_t* sizes, const int32_t* row_ptr, const int32_t* col,
                                            const float* vals, const float* B, int64_t ldb, const float* grad_C,
                                            int64_t ldgc, float* grad_B, int64_t ldgb, float* grad_vals,
                                            int64_t total_rows, int64_t total_nnz) {
  if (!h) return BSPMM_ERROR_INVALID_VALUE;
  if (batch < 0 || k < 1 || ldgc < k || (grad_B && ldgb < k) || (grad_vals && ldb < k) || total_rows < 0 ||
      total_nnz < 0 || total_nnz > INT32_MAX)
    return fail(h, BSPMM_ERROR_INVALID_VALUE, "batch<0, k<1, ld<k or bad totals");
  if (batch == 0 || (!grad_B && !grad_vals)) return BSPMM_SUCCESS;
  if (!row_off || !row_ptr) return fail(h, BSPMM_ERROR_INVALID_VALUE, "NULL pointer argument");
  DeviceGuard g(h->device);
  if (grad_B && grad_vals && !(h->flags & BSPMM_VALIDATE) && !(h->dbg & (2048 | kDbgNoFusedBackward)) &&
      grad_B != grad_C) {
    // streaming batches: one fused kernel (grad_C staged once per matrix,
    // A^T formed in shared memory); other shapes fall through
    bool used = false;
    CK(h, launch_backward_fused(batch, k, row_off, sizes, row_ptr, col, vals, B, ldb, grad_C, ldgc, grad_B, ldgb,
                                grad_vals, h->hint_rows, h->hint_nnz, h->num_sms, h->dbg, h->stream, &used));
    if (used) {
      h->launches++;
      return BSPMM_SUCCESS;
    }
  }
  if (grad_B && grad_vals && !(h->flags & BSPMM_VALIDATE) && !(h->dbg & 2048)) {
    // both adjoints: the transpose (latency-bound) runs on an auxiliary stream
    // concurrently with the SDDMM, then grad_B = A^T grad_C once it has joined
    // (fork / join by events: also valid inside a CUDA-graph capture)
    TransWs w;
    bspmm_status_t st = trans_workspace(h, total_rows, total_nnz, &w);
    if (st != BSPMM_SUCCESS) return st;
    CK(h, cudaEventRecord(h->ev_fork, h->stream));
    CK(h, cudaStreamWaitEvent(h->s_aux, h->ev_fork, 0));
    // from here on every return joins s_aux back into the caller's stream (an
    // unjoined fork would break a graph capture and leave s_aux work unordered)
    struct Join {
      bspmm_handle_t h;
      cudaStream_t main;
      ~Join() {
        h->stream = main;
        cudaEventRecord(h->ev_join, h->s_aux);
        cudaStreamWaitEvent(main, h->ev_join, 0);
      }
    } join{h, h->stream};
    st = transpose_impl(h, batch, row_off, sizes, row_ptr, col, vals, w.rowT, w.colT, w.valsT, h->s_aux);
    if (st != BSPMM_SUCCESS) return st;
    if (!(h->dbg & 4096)) {  // grad_B = A^T grad_C on the auxiliary stream too, after the transpose
      h->stream = h->s_aux;
      st = csr_impl_bwd(h, batch, k, row_off, sizes, w.rowT, w.colT, w.valsT, grad_C, ldgc, grad_B, ldgb);
      h->stream = join.main;
      if (st != BSPMM_SUCCESS) return st;
    }
    st = bspmm_sddmm(h, batch, k, row_off, sizes, row_ptr, col, B, ldb, grad_C, ldgc, grad_vals);
    if (st != BSPMM_SUCCESS) return st;
    if (h->dbg & 4096) {  // grad_B on the caller's stream after the join
      cudaEventRecord(h->ev_join, h->s_aux);
      CK(h, cudaStreamWaitEvent(h->stream, h->ev_join, 0));
      return csr_impl_bwd(h, batch, k, row_off, sizes, w.rowT, w.colT, w.valsT, grad_C, ldgc, grad_B, ldgb);
    }
    return BSPMM_SUCCESS;
  }
  if (grad_vals) {  // dL/dval_e = <grad_C[row_e], B[col_e]>
    bspmm_status_t st = bspmm_sddmm(h, batch, k, row_off, sizes, row_ptr, col, B, ldb, grad_C, ldgc, grad_vals);
    if (st != BSPMM_SUCCESS) return st;
  }
  if (grad_B) {  // dL/dB_i = A_i^T grad_C_i: transpose, then the forward kernel
    TransWs w;
    bspmm_status_t st = trans_workspace(h, total_rows, total_nnz, &w);
    if (st != BSPMM_SUCCESS) return st;
    st = transpose_impl(h, batch, row_off, sizes, row_ptr, col, vals, w.rowT, w.colT, w.valsT);
    if (st != BSPMM_SUCCESS) return st;
    return csr_impl_bwd(h, batch, k, row_off, sizes, w.rowT, w.colT, w.valsT, grad_C, ldgc, grad_B, ldgb);
  }
  return BSPMM_SUCCESS;
}

// ---- end-to-end host-buffer path ------------------------------------------
BSPMM_API bspmm_status_t bspmm_csr_host(bspmm_handle_t h, int32_t batch, int32_t k, const int32_t* sizes_host,
                                        const int32_t* row_ptr_host, const int32_t* col_host,
                                        const float* vals_host, const float* B_host, float* C_host,
                                        int64_t total_rows, int64_t total_nnz) {
  if (!h) return BSPMM_ERROR_INVALID_VALUE;
  if (batch < 0 || k < 1 || total_rows < 0 || total_nnz < 0 || total_nnz > INT32_MAX)
    return fail(h, BSPMM_ERROR_INVALID_VALUE, "batch<0, k<1 or bad totals");
  if (batch == 0) return BSPMM_SUCCESS;
  if (!sizes_host || !row_ptr_host || !B_host || !C_host || (total_nnz > 0 && (!col_host || !vals_host)))
    return fail(h, BSPMM_ERROR_INVALID_VALUE, "NULL pointer argument");
  DeviceGuard g(h->device);
  const int64_t N = total_rows, NNZ = total_nnz;
  // device mirror: [sizes][row_off][row_ptr][col][val][B][C]
  size_t off = 0;
  const size_t o_sz = off; off += al256((size_t)batch * 4);
  const size_t o_ro = off; off += al256((size_t)(batch + 1) * 8);
  const size_t o_rp = off; off += al256((size_t)(N + 1) * 4);
  const size_t o_col = off; off += al256((size_t)NNZ * 4);
  const size_t o_val = off; off += al256((size_t)NNZ * 4);
  const size_t o_B = off; off += al256((size_t)N * k * 4);
  const size_t o_C = off; off += al256((size_t)N * k * 4);
  bspmm_status_t st = grow(h, &h->hbuf, &h->hbuf_bytes, off);
  if (st != BSPMM_SUCCESS) return st;
  char* base = static_cast<char*>(h->hbuf);
  int32_t* d_sz = reinterpret_cast<int32_t*>(base + o_sz);
  int64_t* d_ro = reinterpret_cast<int64_t*>(base + o_ro);
  int32_t* d_rp = reinterpret_cast<int32_t*>(base + o_rp);
  int32_t* d_col = reinterpret_cast<int32_t*>(base + o_col);
  float* d_val = reinterpret_cast<float*>(base + o_val);
  float* d_B = reinterpret_cast<float*>(base + o_B);
  float* d_C = reinterpret_cast<float*>(base + o_C);
  if (!h->s_h2d) CK(h, cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking));
  if (!h->s_d2h) CK(h, cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking));
  for (auto& e : h->ev)
    if (!e) CK(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));

  // chunk plan: contiguous graph ranges of ~equal rows (host arithmetic for scheduling only)
  const int64_t bytesBC = N * (int64_t)k * 4;
  const int nch = (int)std::max<int64_t>(1, std::min<int64_t>(24, (bytesBC + (96 << 20) - 1) / (96 << 20)));
  int32_t gi[25];
  int64_t gr[25];
  gi[0] = 0;
  gr[0] = 0;
  {
    int32_t i = 0;
    int64_t r = 0;
    for (int c = 1; c < nch; ++c) {
      const int64_t target = N * c / nch;
      while (i < batch && r + sizes_host[i] <= target) r += sizes_host[i++];
      gi[c] = i;
      gr[c] = r;
    }
    gi[nch] = batch;
    gr[nch] = N;
  }
  const bool validate = (h->flags & BSPMM_VALIDATE) != 0;
  cudaEvent_t ev_sizes = h->ev[0];
  CK(h, cudaMemcpyAsync(d_sz, sizes_host, (size_t)batch * 4, cudaMemcpyHostToDevice, h->s_h2d));
  CK(h, cudaEventRecord(ev_sizes, h->s_h2d));
  CK(h, cudaStreamWaitEvent(h->stream, ev_sizes, 0));
  st = bspmm_build_offsets(h, batch, d_sz, d_ro);
  if (st != BSPMM_SUCCESS) return st;
  for (int c = 0; c < nch; ++c) {
    const int32_t i0 = gi[c], i1 = gi[c + 1];
    const int64_t r0 = gr[c], r1 = gr[c + 1];
    if (i1 == i0) continue;
    const int64_t z0 = row_ptr_host[r0], z1 = row_ptr_host[r1];
    cudaEvent_t ev_in = h->ev[1 + 2 * c], ev_out = h->ev[2 + 2 * c];
    CK(h, cudaMemcpyAsync(d_rp + r0, row_ptr_host + r0, (size_t)(r1 - r0 + 1) * 4, cudaMemcpyHostToDevice,
                          h->s_h2d));
    if (z1 > z0) {
      CK(h, cudaMemcpyAsync(d_col + z0, col_host + z0, (size_t)(z1 - z0) * 4, cudaMemcpyHostToDevice, h->s_h2d));
      CK(h, cudaMemcpyAsync(d_val + z0, vals_host + z0, (size_t)(z1 - z0) * 4, cudaMemcpyHostToDevice, h->s_h2d));
    }
    CK(h, cudaMemcpyAsync(d_B + r0 * k, B_host + r0 * k, (size_t)(r1 - r0) * k * 4, cudaMemcpyHostToDevice,
                          h->s_h2d));
    CK(h, cudaEventRecord(ev_in, h->s_h2d));
    CK(h, cudaStreamWaitEvent(h->stream, ev_in, 0));
    st = csr_impl(h, i1 - i0, k, d_ro + i0, nullptr, d_rp, d_col, d_val, d_B, k, d_C, k, validate);
    if (st != BSPMM_SUCCESS) return st;
    CK(h, cudaEventRecord(ev_out, h->stream));
    CK(h, cudaStreamWaitEvent(h->s_d2h, ev_out, 0));
    CK(h, cudaMemcpyAsync(C_host + r0 * k, d_C + r0 * k, (size_t)(r1 - r0) * k * 4, cudaMemcpyDeviceToHost,
                          h->s_d2h));
  }
  CK(h, cudaStreamSynchronize(h->s_d2h));
  CK(h, cudaStreamSynchronize(h->stream));
  return BSPMM_SUCCESS;
}

}  // extern "C"
