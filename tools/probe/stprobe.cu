// stprobe.cu — store-phase floor: `ctas` CTAs (one per SM) each write `kb` KB
// of fp32 with 128-bit stores from 480 threads (st.global / st.global.cs),
// cycling over buffers larger than 2x L2 (dirty-line evictions as in a bench).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stprobe stprobe.cu && ./stprobe
#include <cstdio>
#include <cuda_runtime.h>

template <bool CS>
__global__ void st_kernel(float4* out, int per_cta_f4) {
  float4* o = out + (size_t)blockIdx.x * per_cta_f4;
  const float4 v = make_float4(1.f, 2.f, 3.f, (float)blockIdx.x);
  for (int i = threadIdx.x; i < per_cta_f4; i += blockDim.x) {
    if (CS) asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(o + i), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
    else o[i] = v;
  }
}
__global__ void ld_kernel(const float4* in, int per_cta_f4, float* sink) {
  const float4* p = in + (size_t)blockIdx.x * per_cta_f4;
  float acc = 0.f;
  for (int i = threadIdx.x; i < per_cta_f4; i += blockDim.x) { float4 v = __ldcs(p + i); acc += v.x + v.y + v.z + v.w; }
  if (acc == 12345.f) sink[0] = acc;
}

int main() {
  const size_t total = 600ull << 20;
  float4* buf;
  float* sink;
  cudaMalloc(&buf, total);
  cudaMalloc(&sink, 64);
  cudaMemset(buf, 0, total);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int cfgs[][2] = {{100, 100}, {148, 68}, {148, 100}, {100, 50}, {148, 34}};
  for (auto& c : cfgs) {
    const int ctas = c[0], kb = c[1];
    const int per = kb * 1024 / 16;
    const size_t launch_bytes = (size_t)ctas * per * 16;
    const int reps = (int)(total / launch_bytes);
    for (int mode = 0; mode < 3; ++mode) {
      for (int w = 0; w < 2; ++w)
        for (int r = 0; r < reps; ++r) {
          float4* o = buf + (size_t)r * ctas * per;
          if (mode == 0) st_kernel<false><<<ctas, 480>>>(o, per);
          else if (mode == 1) st_kernel<true><<<ctas, 480>>>(o, per);
          else ld_kernel<<<ctas, 480>>>(o, per, sink);
        }
      cudaEventRecord(a);
      for (int r = 0; r < reps; ++r) {
        float4* o = buf + (size_t)r * ctas * per;
        if (mode == 0) st_kernel<false><<<ctas, 480>>>(o, per);
        else if (mode == 1) st_kernel<true><<<ctas, 480>>>(o, per);
        else ld_kernel<<<ctas, 480>>>(o, per, sink);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double us = ms * 1e3 / reps;
      printf("ctas %3d x %3d KB  %-8s  %6.2f us/launch  %6.0f GB/s\n", ctas, kb,
             mode == 0 ? "st" : mode == 1 ? "st.cs" : "ld.cs", us, launch_bytes / us / 1e3);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
