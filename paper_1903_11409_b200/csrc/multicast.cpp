// multicast.cpp — NVSwitch multicast buffers for the all-gather fused into the
// SpMM store (SURVEY §8(e) optional reassembly, §8(f) NEXT-4b).
//
// A team of G GPUs (one process each, or one process with G=1) shares one
// multicast object.  Every member binds a physical buffer of its own device to
// it and maps two virtual ranges: the UNICAST range (its own copy of C, read
// with ordinary loads) and the MULTICAST range (a store there lands in the
// bound buffer of every member).  bspmm_csr_multicast writes each rank's
// shard of C through the multicast range, so the full C appears on every GPU
// without a separate collective launch.
//
// Driver entry points are fetched through the runtime (no link-time libcuda).
// Handle exchange between processes: the root exports a POSIX file descriptor
// (bspmm_mc_create), the caller passes it to the other ranks (SCM_RIGHTS over
// a Unix socket, paper_1903_11409_b200/dist.py) and they bspmm_mc_import it.
// Protocol: create/import (each adds its own device) -> barrier over the team
// -> bspmm_mc_bind on every rank -> barrier -> use.
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <string>

#include "bspmm.h"

namespace {

struct Driver {
  decltype(&cuMulticastCreate) mcCreate = nullptr;
  decltype(&cuMulticastAddDevice) mcAddDevice = nullptr;
  decltype(&cuMulticastBindMem) mcBindMem = nullptr;
  decltype(&cuMulticastUnbind) mcUnbind = nullptr;
  decltype(&cuMulticastGetGranularity) mcGranularity = nullptr;
  decltype(&cuMemCreate) memCreate = nullptr;
  decltype(&cuMemRelease) memRelease = nullptr;
  decltype(&cuMemAddressReserve) addrReserve = nullptr;
  decltype(&cuMemAddressFree) addrFree = nullptr;
  decltype(&cuMemMap) memMap = nullptr;
  decltype(&cuMemUnmap) memUnmap = nullptr;
  decltype(&cuMemSetAccess) memSetAccess = nullptr;
  decltype(&cuMemGetAllocationGranularity) memGranularity = nullptr;
  decltype(&cuMemExportToShareableHandle) memExport = nullptr;
  decltype(&cuMemImportFromShareableHandle) memImport = nullptr;
  decltype(&cuDeviceGet) deviceGet = nullptr;
  decltype(&cuDeviceGetAttribute) deviceGetAttribute = nullptr;
  bool ok = false;
};

template <typename F>
bool fetch(const char* name, F* out) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn) {
    cudaGetLastError();
    return false;
  }
  *out = reinterpret_cast<F>(fn);
  return true;
}

const Driver& drv() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    d.ok = fetch("cuMulticastCreate", &d.mcCreate) && fetch("cuMulticastAddDevice", &d.mcAddDevice) &&
           fetch("cuMulticastBindMem", &d.mcBindMem) && fetch("cuMulticastUnbind", &d.mcUnbind) &&
           fetch("cuMulticastGetGranularity", &d.mcGranularity) && fetch("cuMemCreate", &d.memCreate) &&
           fetch("cuMemRelease", &d.memRelease) && fetch("cuMemAddressReserve", &d.addrReserve) &&
           fetch("cuMemAddressFree", &d.addrFree) && fetch("cuMemMap", &d.memMap) &&
           fetch("cuMemUnmap", &d.memUnmap) && fetch("cuMemSetAccess", &d.memSetAccess) &&
           fetch("cuMemGetAllocationGranularity", &d.memGranularity) &&
           fetch("cuMemExportToShareableHandle", &d.memExport) &&
           fetch("cuMemImportFromShareableHandle", &d.memImport) && fetch("cuDeviceGet", &d.deviceGet) &&
           fetch("cuDeviceGetAttribute", &d.deviceGetAttribute);
  });
  return d;
}

size_t round_up(size_t x, size_t g) { return (x + g - 1) / g * g; }

thread_local std::string g_err;

// record which driver call failed (bspmm_mc_last_error)
bool ck(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return true;
  char buf[160];
  snprintf(buf, sizeof buf, "%s failed: CUresult %d", what, (int)r);
  g_err = buf;
  return false;
}

}  // namespace

struct bspmm_mc_s {
  int device = 0;
  int num_devices = 1;
  size_t bytes = 0;  // rounded to the multicast granularity
  CUmemGenericAllocationHandle mc = 0, mem = 0;
  CUdeviceptr uc_va = 0, mc_va = 0;
  bool have_mc = false, have_mem = false, bound = false, uc_mapped = false, mc_mapped = false;
  bool uc_reserved = false, mc_reserved = false;
};

// the mc_* entry points switch to the object's device and restore the caller's
struct McDeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit McDeviceGuard(int d) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != d) ok = cudaSetDevice(d) == cudaSuccess;
  }
  ~McDeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

extern "C" {

BSPMM_API int32_t bspmm_mc_supported(int device) {
  const Driver& d = drv();
  if (!d.ok) return 0;
  cudaFree(nullptr);  // make sure a context exists
  CUdevice dev;
  if (d.deviceGet(&dev, device) != CUDA_SUCCESS) return 0;
  int v = 0;
  if (d.deviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS) return 0;
  return v ? 1 : 0;
}

static bspmm_status_t mc_prop(int num_devices, size_t bytes, CUmulticastObjectProp* prop, size_t* rounded) {
  const Driver& d = drv();
  *prop = {};
  prop->numDevices = (unsigned)num_devices;
  prop->handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  prop->size = bytes;
  size_t g = 0;
  if (!ck(d.mcGranularity(&g, prop, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity") || g == 0)
    return BSPMM_ERROR_CUDA;
  *rounded = round_up(bytes, g);
  prop->size = *rounded;
  return BSPMM_SUCCESS;
}

static bspmm_status_t add_self(bspmm_mc_s* m) {
  const Driver& d = drv();
  CUdevice dev;
  if (!ck(d.deviceGet(&dev, m->device), "cuDeviceGet")) return BSPMM_ERROR_CUDA;
  if (!ck(d.mcAddDevice(m->mc, dev), "cuMulticastAddDevice")) return BSPMM_ERROR_CUDA;
  return BSPMM_SUCCESS;
}

BSPMM_API bspmm_status_t bspmm_mc_destroy(bspmm_mc_t m);

BSPMM_API bspmm_status_t bspmm_mc_create(int device, int num_devices, size_t bytes, int exportable,
                                         bspmm_mc_t* out, int* fd_out) {
  if (!out || num_devices < 1 || bytes == 0 || (exportable && !fd_out)) return BSPMM_ERROR_INVALID_VALUE;
  *out = nullptr;
  if (!bspmm_mc_supported(device)) return BSPMM_ERROR_NOT_SUPPORTED;
  const Driver& d = drv();
  McDeviceGuard dg(device);
  if (!dg.ok) return BSPMM_ERROR_CUDA;
  bspmm_mc_s* m = new bspmm_mc_s;
  m->device = device;
  m->num_devices = num_devices;
  CUmulticastObjectProp prop;
  bspmm_status_t st = mc_prop(num_devices, bytes, &prop, &m->bytes);
  if (st == BSPMM_SUCCESS && !ck(d.mcCreate(&m->mc, &prop), "cuMulticastCreate")) st = BSPMM_ERROR_CUDA;
  if (st == BSPMM_SUCCESS) m->have_mc = true;
  if (st == BSPMM_SUCCESS && exportable) {
    int fd = -1;
    if (!ck(d.memExport(&fd, m->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "cuMemExportToShareableHandle"))
      st = BSPMM_ERROR_CUDA;
    else *fd_out = fd;
  }
  if (st == BSPMM_SUCCESS) st = add_self(m);
  if (st != BSPMM_SUCCESS) {
    bspmm_mc_destroy(m);
    return st;
  }
  *out = m;
  return BSPMM_SUCCESS;
}

BSPMM_API bspmm_status_t bspmm_mc_import(int device, int num_devices, size_t bytes, int fd, bspmm_mc_t* out) {
  if (!out || num_devices < 1 || bytes == 0 || fd < 0) return BSPMM_ERROR_INVALID_VALUE;
  *out = nullptr;
  if (!bspmm_mc_supported(device)) return BSPMM_ERROR_NOT_SUPPORTED;
  const Driver& d = drv();
  McDeviceGuard dg(device);
  if (!dg.ok) return BSPMM_ERROR_CUDA;
  bspmm_mc_s* m = new bspmm_mc_s;
  m->device = device;
  m->num_devices = num_devices;
  CUmulticastObjectProp prop;
  bspmm_status_t st = mc_prop(num_devices, bytes, &prop, &m->bytes);
  if (st == BSPMM_SUCCESS &&
      !ck(d.memImport(&m->mc, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)),
                      CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
          "cuMemImportFromShareableHandle"))
    st = BSPMM_ERROR_CUDA;
  if (st == BSPMM_SUCCESS) m->have_mc = true;
  if (st == BSPMM_SUCCESS) st = add_self(m);
  if (st != BSPMM_SUCCESS) {
    bspmm_mc_destroy(m);
    return st;
  }
  *out = m;
  return BSPMM_SUCCESS;
}

BSPMM_API bspmm_status_t bspmm_mc_bind(bspmm_mc_t m, void** uc_ptr, void** mc_ptr) {
  if (!m || !uc_ptr || !mc_ptr) return BSPMM_ERROR_INVALID_VALUE;
  const Driver& d = drv();
  McDeviceGuard dg(m->device);
  if (!dg.ok) return BSPMM_ERROR_CUDA;
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = m->device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_NONE;
  size_t g = 0;
  if (!ck(d.memGranularity(&g, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity") || g == 0)
    return BSPMM_ERROR_CUDA;
  if (m->bytes % g) return BSPMM_ERROR_NOT_SUPPORTED;
  if (!ck(d.memCreate(&m->mem, m->bytes, &ap, 0), "cuMemCreate")) return BSPMM_ERROR_OUT_OF_MEMORY;
  m->have_mem = true;
  if (!ck(d.mcBindMem(m->mc, 0, m->mem, 0, m->bytes, 0), "cuMulticastBindMem")) return BSPMM_ERROR_CUDA;
  m->bound = true;
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = m->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (!ck(d.addrReserve(&m->uc_va, m->bytes, g, 0, 0), "cuMemAddressReserve(uc)")) return BSPMM_ERROR_CUDA;
  m->uc_reserved = true;
  if (!ck(d.memMap(m->uc_va, m->bytes, 0, m->mem, 0), "cuMemMap(uc)")) return BSPMM_ERROR_CUDA;
  m->uc_mapped = true;
  if (!ck(d.memSetAccess(m->uc_va, m->bytes, &acc, 1), "cuMemSetAccess(uc)")) return BSPMM_ERROR_CUDA;
  if (!ck(d.addrReserve(&m->mc_va, m->bytes, g, 0, 0), "cuMemAddressReserve(mc)")) return BSPMM_ERROR_CUDA;
  m->mc_reserved = true;
  if (!ck(d.memMap(m->mc_va, m->bytes, 0, m->mc, 0), "cuMemMap(mc)")) return BSPMM_ERROR_CUDA;
  m->mc_mapped = true;
  if (!ck(d.memSetAccess(m->mc_va, m->bytes, &acc, 1), "cuMemSetAccess(mc)")) return BSPMM_ERROR_CUDA;
  *uc_ptr = reinterpret_cast<void*>(m->uc_va);
  *mc_ptr = reinterpret_cast<void*>(m->mc_va);
  return BSPMM_SUCCESS;
}

BSPMM_API const char* bspmm_mc_last_error(void) { return g_err.c_str(); }

BSPMM_API size_t bspmm_mc_bytes(bspmm_mc_t m) { return m ? m->bytes : 0; }

BSPMM_API bspmm_status_t bspmm_mc_destroy(bspmm_mc_t m) {
  if (!m) return BSPMM_SUCCESS;
  const Driver& d = drv();
  McDeviceGuard dg(m->device);
  // the team buffer may be in use by work on any of the caller's streams,
  // which the object does not know: drain the device before unmapping
  cudaDeviceSynchronize();
  if (m->mc_mapped) d.memUnmap(m->mc_va, m->bytes);
  if (m->mc_reserved) d.addrFree(m->mc_va, m->bytes);
  if (m->uc_mapped) d.memUnmap(m->uc_va, m->bytes);
  if (m->uc_reserved) d.addrFree(m->uc_va, m->bytes);
  if (m->bound) {
    CUdevice dev;
    if (d.deviceGet(&dev, m->device) == CUDA_SUCCESS) d.mcUnbind(m->mc, dev, 0, m->bytes);
  }
  if (m->have_mem) d.memRelease(m->mem);
  if (m->have_mc) d.memRelease(m->mc);
  delete m;
  return BSPMM_SUCCESS;
}

}  // extern "C"
