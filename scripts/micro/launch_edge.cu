// Microbenchmark: the event-timed cost of an (almost) empty launch shaped like the maintenance
// kernel (296 blocks x 512 threads, ~110 KB dynamic shared memory), cooperative or not, right
// after a busy kernel that uses a different shared-memory footprint.  Separates launch/drain
// edges from the maintenance kernel's own work.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/micro/launch_edge.cu -o /tmp/launch_edge
#include <cstdio>
#include <cuda_runtime.h>

__global__ void busy(float* out, int iters) {
  extern __shared__ float sm[];
  float a = threadIdx.x;
  for (int i = 0; i < iters; ++i) a = a * 0.999f + 0.001f;
  sm[threadIdx.x] = a;
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sm[(threadIdx.x + 1) % blockDim.x];
}
__global__ void __launch_bounds__(512, 2) empty_k(int* flag, int4* dst, const int4* src, int rows) {
  extern __shared__ int4 s_rows[];
  // optional copy work: rows x 512 B per block through shared memory
  for (int r = 0; r < rows; ++r) {
    const long long o = ((long long)blockIdx.x * rows + r) * 32;
    if (threadIdx.x < 32) s_rows[r * 32 + threadIdx.x] = src[o + threadIdx.x];
  }
  __syncthreads();
  for (int r = 0; r < rows; ++r) {
    const long long o = ((long long)blockIdx.x * rows + r) * 32;
    if (threadIdx.x < 32) dst[o + threadIdx.x] = s_rows[r * 32 + threadIdx.x];
  }
  if (threadIdx.x == 0 && blockIdx.x == 0 && flag) *flag = 1;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, (size_t)sms * 4 * 1024 * 4);
  int* flag; cudaMalloc(&flag, 4);
  const int maxrows = 210;
  int4 *src, *dst;
  cudaMalloc(&src, (size_t)2 * sms * maxrows * 512);
  cudaMalloc(&dst, (size_t)2 * sms * maxrows * 512);
  cudaMemset(src, 1, (size_t)2 * sms * maxrows * 512);
  const int smem_e = 110 * 1024;
  cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_e);
  cudaFuncSetAttribute(busy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
  for (int busy_smem : {4 * 1024, 200 * 1024}) {
    for (int coop = 0; coop < 2; ++coop) {
      for (int rows : {0, 56, 112, 210}) {
        float tot = 0.f, totb = 0.f;
        const int reps = 50;
        for (int rep = 0; rep < reps + 5; ++rep) {
          busy<<<sms, 512, busy_smem>>>(out, 20000);
          cudaEventRecord(e0);
          int* f = flag;
          int4* d = dst; const int4* s = src; int r = rows;
          void* args[] = {&f, &d, &s, &r};
          if (coop)
            cudaLaunchCooperativeKernel((void*)empty_k, dim3(2 * sms), dim3(512), args, smem_e, 0);
          else
            empty_k<<<2 * sms, 512, smem_e>>>(flag, dst, src, rows);
          cudaEventRecord(e1);
          empty_k<<<2 * sms, 512, smem_e>>>(flag, dst, src, 0);
          cudaEventRecord(e2);
          cudaEventSynchronize(e2);
          float ms = 0.f, ms2 = 0.f;
          cudaEventElapsedTime(&ms, e0, e1);
          cudaEventElapsedTime(&ms2, e1, e2);
          if (rep >= 5) { tot += ms; totb += ms2; }
        }
        const double bytes = 2.0 * 2 * sms * rows * 512;
        printf("busy smem %3d KB  %s  rows %3d: after-busy %7.2f us (%6.2f TB/s)   back-to-back empty %6.2f us  (%s)\n",
               busy_smem / 1024, coop ? "coop    " : "non-coop", rows, tot / reps * 1e3,
               rows ? bytes / (tot / reps * 1e-3) / 1e12 : 0.0, totb / reps * 1e3,
               cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  // empty launches of other shapes, back to back (event to event)
  struct Shape { int blocks, threads, smem; };
  for (Shape sh : {Shape{1, 32, 0}, Shape{148, 128, 0}, Shape{148, 512, 0}, Shape{296, 512, 0},
                   Shape{296, 256, 0}, Shape{296, 512, 48 * 1024}, Shape{296, 512, 110 * 1024},
                   Shape{148, 1024, 0}, Shape{148, 512, 220 * 1024}}) {
    if (sh.smem > 110 * 1024)
      cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, sh.smem);
    float tot = 0.f;
    for (int rep = 0; rep < 105; ++rep) {
      cudaEventRecord(e1);
      empty_k<<<sh.blocks, sh.threads, sh.smem>>>(flag, dst, src, 0);
      cudaEventRecord(e2);
      cudaEventSynchronize(e2);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e1, e2);
      if (rep >= 5) tot += ms;
    }
    printf("empty %4d blocks x %4d threads, %3d KB smem: %6.2f us  (%s)\n", sh.blocks, sh.threads,
           sh.smem / 1024, tot / 100 * 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  // two empty launches between one event pair: the per-launch increment
  {
    float tot = 0.f;
    for (int rep = 0; rep < 105; ++rep) {
      cudaEventRecord(e1);
      for (int k = 0; k < 10; ++k) empty_k<<<296, 512, 110 * 1024>>>(flag, dst, src, 0);
      cudaEventRecord(e2);
      cudaEventSynchronize(e2);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e1, e2);
      if (rep >= 5) tot += ms;
    }
    printf("10 empty 296x512 110KB launches in one event pair: %6.2f us each\n", tot / 100 * 1e3 / 10);
  }
  return 0;
}
