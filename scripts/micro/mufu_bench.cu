// Microbenchmark: MUFU ex2 and FFMA / FFMA2 throughput per SM per clock on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void ex2_kernel(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f - 3.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i])); a[i] = y - 3.f; }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ffma_kernel(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], 0.999f, 0.001f);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ffma2_kernel(float* out, int iters) {
  float2 a[8];
  for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  const float2 m = make_float2(0.999f, 0.999f), c = make_float2(0.001f, 0.001f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], m, c);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, sms * 8 * 1024 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096;
  for (int k = 0; k < 3; ++k) {
    for (int warm = 0; warm < 2; ++warm) {
      cudaEventRecord(a);
      if (k == 0) ex2_kernel<<<sms * 4, 512>>>(out, iters);
      if (k == 1) ffma_kernel<<<sms * 4, 512>>>(out, iters);
      if (k == 2) ffma2_kernel<<<sms * 4, 512>>>(out, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double ops = (double)sms * 4 * 512 * iters * 8 * (k == 2 ? 2 : 1);
      if (warm) printf("%s: %.3f ms, %.2f Gop/s, %.2f lane-ops/clk/SM at %d MHz (max clock)\n",
                       k == 0 ? "ex2" : (k == 1 ? "ffma" : "ffma2(lanes x2)"), ms, ops / ms / 1e6,
                       ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
