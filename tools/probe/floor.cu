// floor.cu — copy floors for the small-batch configs (NOT product code; a
// measurement probe for tools/kbench.py --copy-baseline).  A hand-written copy
// of the same B bytes into C, spread evenly over one CTA per SM and launched
// exactly like the SpMM kernels (programmatic stream serialization, inside the
// same CUDA graph): what moving the batch's dense bytes costs with no metadata
// and no arithmetic.  mode & 3:
//   0: cp.async 16 B -> shared memory in G groups on mbarriers, each group
//      stored (st.global.cs.v4) as it lands -- the spread kernel's data path;
//   1: ld.global.nc.v4 -> registers -> st.global.cs.v4, all loads first;
//   2: TMA 1-D bulk copies (G chunks, one mbarrier each) -> threads store;
//   3: TMA 1-D bulk loads + TMA bulk stores (shared -> global) per chunk.
// mode & 4: a dependent round trip first (every thread loads dep[blockIdx.x]
//   and branches on it before touching B: the SpMM's row-offset read);
// mode & 8: that load with an L2 evict_last policy.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o libfloor.so floor.cu
#include <cstdint>
#include <cuda_runtime.h>

namespace {
constexpr int kThreads = 1024;
__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void wait_bar(uint64_t* b) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(sa(b)) : "memory");
}
__device__ __forceinline__ void stcs(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ bool dep_rt(const int64_t* dep, int mode) {
  if (!(mode & 4)) return false;
  int64_t v;
  if (mode & 8) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.nc.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(dep + blockIdx.x % 64), "l"(pol));
  } else {
    v = dep[blockIdx.x % 64];
  }
  return v == -123456789;  // never: a control dependence on the loaded value
}

__global__ void __launch_bounds__(kThreads, 1) copy_k(const float4* __restrict__ B, float4* __restrict__ C,
                                                      int64_t n4, int groups, int mode, const int64_t* dep) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  float4* S = reinterpret_cast<float4*>(smem + 128);
  const int method = mode & 3;
  if (threadIdx.x == 0 && method != 1) {
    for (int g = 0; g < groups; ++g)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar[g])), "r"(method == 0 ? kThreads : 1)
                   : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (dep_rt(dep, mode)) return;
  const int64_t lo = n4 * blockIdx.x / gridDim.x, hi = n4 * (blockIdx.x + 1) / gridDim.x;
  const int32_t cnt = (int32_t)(hi - lo);
  if (method == 1) {
    constexpr int U = 8;
    for (int64_t q0 = lo + threadIdx.x; q0 < hi; q0 += (int64_t)U * kThreads) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t q = q0 + (int64_t)u * kThreads;
        if (q < hi) v[u] = __ldg(B + q);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t q = q0 + (int64_t)u * kThreads;
        if (q < hi) stcs(C + q, v[u]);
      }
    }
    return;
  }
  if (method == 0) {
    for (int g = 0; g < groups; ++g) {
      const int32_t a = cnt * g / groups, b = cnt * (g + 1) / groups;
      for (int32_t q = a + threadIdx.x; q < b; q += kThreads)
        asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(sa(S + q)), "l"(B + lo + q) : "memory");
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(&bar[g])) : "memory");
    }
  } else if (threadIdx.x < groups) {  // TMA: chunk g by lane g
    const int g = threadIdx.x;
    const int32_t a = cnt * g / groups, b = cnt * (g + 1) / groups;
    const uint32_t bytes = (uint32_t)(b - a) * 16u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[g])), "r"(bytes) : "memory");
    if (bytes)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(S + a)), "l"(B + lo + a), "r"(bytes), "r"(sa(&bar[g])) : "memory");
  }
  for (int g = 0; g < groups; ++g) {
    const int32_t a = cnt * g / groups, b = cnt * (g + 1) / groups;
    if (method == 3) {
      if (threadIdx.x == g) {
        wait_bar(&bar[g]);
        if (b > a)
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(C + lo + a), "r"(sa(S + a)),
                       "r"((uint32_t)(b - a) * 16u) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      continue;
    }
    wait_bar(&bar[g]);
    for (int32_t q = a + threadIdx.x; q < b; q += kThreads) stcs(C + lo + q, S[q]);
  }
}
}  // namespace

extern "C" int floor_copy(const void* B, void* C, int64_t n4, int mode, int groups, int grid, void* stream,
                          const void* dep) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (groups < 1 || groups > 16) return -2;
  const int64_t per = (n4 + grid - 1) / grid;
  const int smem = (mode & 3) == 1 ? 0 : (int)(128 + per * 16);
  if (smem > 232448 - 1024) return -1;
  cudaFuncSetAttribute(copy_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem > 0 ? smem : 0);
  cfg.dynamicSmemBytes = smem;
  return (int)cudaLaunchKernelEx(&cfg, copy_k, static_cast<const float4*>(B), static_cast<float4*>(C), n4, groups,
                                 mode, static_cast<const int64_t*>(dep));
}
