// opcost.cu — issue cost (SM clock cycles) of the producer's instructions on
// sm_100a, one warp, measured with clock64 around each op.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o opcost opcost.cu && ./opcost
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void k(const float* __restrict__ src, unsigned long long* out, unsigned long long* sink) {
  __shared__ __align__(128) float buf[8192];
  __shared__ __align__(8) uint64_t bar[4];
  const int lane = threadIdx.x;
  if (lane == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar[i])), "r"(32));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  long long t0, t1;
  int k = 0;
#define MEAS(code)                                   \
  __syncwarp();                                      \
  t0 = clock64();                                    \
  code;                                              \
  __syncwarp();                                      \
  t1 = clock64();                                    \
  if (lane == 0) out[blockIdx.x * 16 + k] = t1 - t0; \
  ++k;
  unsigned long long g = 0;
  MEAS(g += gt());                                        // 0 globaltimer (first)
  MEAS(g += gt());                                        // 1 globaltimer (second)
  MEAS(if (lane == 0) sink[blockIdx.x] = g);              // 2 STG one lane
  MEAS(asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&bar[0])) : "memory"));  // 3 arrive x32
  MEAS(asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(&bar[1])) : "memory"));  // 4 noinc
  uint32_t ok = 0;
  MEAS(asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(sa(&bar[2])), "r"(1u) : "memory"));  // 5 try_wait fresh parity 1
  int v = lane;
  MEAS(v = __shfl_sync(0xffffffffu, v, 3));               // 6 shfl
  MEAS(asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(&buf[lane * 4])), "l"(src + lane * 4) : "memory"));  // 7 LDGSTS 16 (cold)
  MEAS(asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(&buf[512 + lane * 4])), "l"(src + 4096 + lane * 4) : "memory"));  // 8 LDGSTS 16 (2nd)
  MEAS(asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa(&buf[1024 + lane])), "l"(src + 8192 + lane) : "memory"));  // 9 LDGSTS 4
  MEAS(if (lane == 0) asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar[3])), "r"(4096u) : "memory"));  // 10 expect_tx
  MEAS(if (lane == 0) asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(&buf[2048])), "l"(src + 16384), "r"(4096u), "r"(sa(&bar[3])) : "memory"));  // 11 bulk copy (cold)
  MEAS(if (lane == 1) asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(&buf[3072])), "l"(src + 20480), "r"(4096u), "r"(sa(&bar[3])) : "memory"));  // 12 bulk copy (2nd)
  MEAS(v += (int)__ldg(src + 32768 + lane));               // 13 LDG (dependent use)
  MEAS(v += (int)__ldg(src + 32768 + 64 + lane));          // 14 LDG same line region (L1/L2 hit)
  if (lane == 0 && v == 12345 && ok == 7) sink[0] = 1;
}

int main() {
  float* src;
  unsigned long long *out, *sink;
  cudaMalloc(&src, 64 << 20);
  cudaMemset(src, 0, 64 << 20);
  cudaMalloc(&out, 148 * 16 * 8);
  cudaMalloc(&sink, 148 * 8);
  const char* names[] = {"globaltimer#1", "globaltimer#2", "stg", "mbar.arrive", "cp.async.arrive.noinc",
                         "try_wait(fresh)", "shfl", "ldgsts16 cold", "ldgsts16 2nd", "ldgsts4", "expect_tx",
                         "bulk 4KB cold", "bulk 4KB 2nd", "ldg+use cold", "ldg+use near"};
  for (int rep = 0; rep < 3; ++rep) {
    k<<<148, 32>>>(src + rep * 65536, out, sink);
    cudaDeviceSynchronize();
    unsigned long long h[148 * 16];
    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
    printf("rep %d (cycles, median over 148 CTAs):\n", rep);
    for (int i = 0; i < 15; ++i) {
      unsigned long long v[148];
      for (int b = 0; b < 148; ++b) v[b] = h[b * 16 + i];
      for (int a = 0; a < 148; ++a)
        for (int b = a + 1; b < 148; ++b)
          if (v[b] < v[a]) { unsigned long long t = v[a]; v[a] = v[b]; v[b] = t; }
      printf("  %-22s %8llu  (min %llu max %llu)\n", names[i], v[74], v[0], v[147]);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
