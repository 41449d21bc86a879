// streamprobe.cu — read-only TMA streaming patterns at C5's SDDMM volume (NOT
// product code): does the order in which the CTAs sweep the operands, or
// reading two operands at once, change the HBM read bandwidth?
//   mode 0: CTA b reads its own contiguous range (bwprobe's pattern)
//   mode 1: front sweep -- chunk j of the array goes to CTA j % grid
//   mode 2: front sweep over TWO arrays (chunk j of A, then chunk j of B)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o streamprobe streamprobe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void stream(const char* A, const char* Bv, size_t total, int chunk, int stages, int mode, float* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[16];
  if (threadIdx.x != 0) return;
  const size_t nchunks = total / chunk;
  size_t my = 0;
  for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  // the list of this CTA's copies: (array, offset)
  const size_t G = gridDim.x;
  size_t count;
  if (mode == 0) count = nchunks / G;
  else if (mode == 1) count = (nchunks + G - 1 - blockIdx.x) / G;
  else count = 2 * ((nchunks + G - 1 - blockIdx.x) / G);
  for (size_t j = 0; j < count; ++j) {
    const char* src;
    if (mode == 0) src = A + ((size_t)blockIdx.x * (nchunks / G) + j) * chunk;
    else if (mode == 1) src = A + (j * G + blockIdx.x) * chunk;
    else src = ((j & 1) ? Bv : A) + ((j >> 1) * G + blockIdx.x) * chunk;
    const int s = (int)(j % stages);
    if (j >= (size_t)stages) {
      const uint32_t ph = ((j / stages) - 1) & 1;
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(ok) : "r"(sa(&bar[s])), "r"(ph) : "memory");
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(sm + (size_t)s * chunk)), "l"(src), "r"(chunk), "r"(sa(&bar[s])) : "memory");
    my += chunk;
  }
  for (size_t j = count > (size_t)stages ? count - stages : 0; j < count; ++j) {
    const int s = (int)(j % stages);
    const uint32_t ph = (j / stages) & 1;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(sa(&bar[s])), "r"(ph) : "memory");
  }
  sink[blockIdx.x] = (float)sm[0] + (float)my;
}

int main() {
  const size_t total = (size_t)2680 << 20;  // one C5 operand (2.68 GB)
  char *A, *Bv;
  float* sink;
  cudaMalloc(&A, total);
  cudaMalloc(&Bv, total);
  cudaMalloc(&sink, 4096 * 4);
  cudaMemset(A, 1, total);
  cudaMemset(Bv, 1, total);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode : {0, 1, 2}) {
    for (int chunk : {16384, 40960}) {
      for (int stages : {2, 4, 5}) {
        if ((size_t)chunk * stages > 220 * 1024) continue;
        auto go = [&] { stream<<<sms, 32, (size_t)chunk * stages>>>(A, Bv, total, chunk, stages, mode, sink); };
        go();
        cudaEventRecord(a);
        for (int r = 0; r < 3; ++r) go();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)(total / chunk) * chunk * (mode == 2 ? 2 : 1) * 3;
        printf("{\"mode\": %d, \"chunk_KB\": %d, \"stages\": %d, \"inflight_KB\": %d, \"GBs\": %.1f, \"err\": \"%s\"}\n",
               mode, chunk / 1024, stages, chunk * stages / 1024, bytes / (ms * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
