// bwprobe.cu — calibrates per-SM HBM read (and write) bandwidth on B200 for
// the two paths the SpMM kernel can use: TMA bulk copies into shared memory
// (one issuing thread, S buffers in flight) and LSU 128-bit loads (all warps).
// Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bwprobe bwprobe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void tma_read(const char* src, size_t per_cta, int chunk, int stages, float* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[16];
  const char* base = src + (size_t)blockIdx.x * per_cta;
  const int n = (int)(per_cta / chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    for (int j = 0; j < n; ++j) {
      const int s = j % stages;
      if (j >= stages) {  // wait for the copy that used this buffer
        const uint32_t ph = ((j / stages) - 1) & 1;
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(sa(&bar[s])), "r"(ph) : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sa(sm + (size_t)s * chunk)), "l"(base + (size_t)j * chunk), "r"(chunk), "r"(sa(&bar[s])) : "memory");
    }
    for (int j = n > stages ? n - stages : 0; j < n; ++j) {
      const int s = j % stages;
      const uint32_t ph = (j / stages) & 1;
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(ok) : "r"(sa(&bar[s])), "r"(ph) : "memory");
    }
    sink[blockIdx.x] = (float)sm[0];
  }
}

template <int U>
__global__ void lsu_read(const float4* src, size_t per_cta_f4, float* sink) {
  const float4* base = src + (size_t)blockIdx.x * per_cta_f4;
  float acc = 0.f;
  for (size_t i = threadIdx.x; i < per_cta_f4; i += (size_t)blockDim.x * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t q = i + (size_t)u * blockDim.x;
      v[u] = q < per_cta_f4 ? __ldcs(base + q) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1.2345f) sink[blockIdx.x] = acc;
}

__global__ void lsu_copy(const float4* src, float4* dst, size_t per_cta_f4) {
  const size_t o = (size_t)blockIdx.x * per_cta_f4;
  for (size_t i = threadIdx.x; i < per_cta_f4; i += blockDim.x) __stcs(dst + o + i, __ldcs(src + o + i));
}

int main() {
  const size_t total = (size_t)1 << 31;  // 2 GiB read
  char* src;
  char* dst;
  float* sink;
  cudaMalloc(&src, total);
  cudaMalloc(&dst, total);
  cudaMalloc(&sink, 4096 * 4);
  cudaMemset(src, 1, total);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(tma_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  auto run = [&](auto launch, const char* name, double bytes) {
    launch();
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"probe\": \"%s\", \"GBs\": %.1f, \"err\": \"%s\"}\n", name, bytes * 5 / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
  };
  for (int ctas_per_sm : {1, 2}) {
    const int grid = sms * ctas_per_sm;
    const size_t per = total / grid / 65536 * 65536;
    for (int chunk : {8192, 16384, 32768, 65536}) {
      for (int stages : {1, 2, 3, 4, 6}) {
        if ((size_t)chunk * stages > (ctas_per_sm == 1 ? 200u : 100u) * 1024) continue;
        char name[128];
        snprintf(name, sizeof name, "tma grid=%d chunk=%dK stages=%d inflight=%dK/SM", grid, chunk / 1024, stages,
                 chunk * stages * ctas_per_sm / 1024);
        run([&] { tma_read<<<grid, 32, (size_t)chunk * stages>>>(src, per, chunk, stages, sink); }, name,
            (double)per * grid);
      }
    }
  }
  for (int threads : {256, 512, 1024}) {
    const int grid = sms;
    const size_t per = total / grid / 16 / 16 * 16;
    char name[128];
    snprintf(name, sizeof name, "lsu_read grid=%d threads=%d unroll=4", grid, threads);
    run([&] { lsu_read<4><<<grid, threads>>>((const float4*)src, per, sink); }, name, (double)per * 16 * grid);
    snprintf(name, sizeof name, "lsu_copy grid=%d threads=%d (read+write)", grid, threads);
    run([&] { lsu_copy<<<grid, threads>>>((const float4*)src, (float4*)dst, per); }, name, 2.0 * per * 16 * grid);
  }
  {
    const int grid = sms * 8;
    const size_t per = total / grid / 16 / 16 * 16;
    run([&] { lsu_copy<<<grid, 256>>>((const float4*)src, (float4*)dst, per); }, "lsu_copy grid=8xSM threads=256 (read+write)",
        2.0 * per * 16 * grid);
  }
  return 0;
}
