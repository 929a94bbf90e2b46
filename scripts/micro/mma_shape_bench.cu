// Microbenchmark: tcgen05.mma bf16 -> fp32 throughput per instruction shape on this B200, one
// CTA per SM, one thread issuing back-to-back MMAs (operands resident, no TMA).  Answers "what
// fraction of the cuBLAS-measured peak can a single-CTA M = 128 kernel reach for the shapes
// attention uses (QK^T: N = 128 keys, A = Q from TMEM or shared memory; PV: N = d = 128)".
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2406_17808_b200/csrc \
//        scripts/micro/mma_shape_bench.cu -o /tmp/mma_shape_bench -lcuda
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_util.cuh"
using namespace cascade;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_bench(int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                  // 128 x 64 bf16 (K-major SW128) x 2 blocks
  uint8_t* sB = smem + 32768;          // N x 64 x 2 blocks
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < (32768 + N * 256) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if ((threadIdx.x >> 5) == 0) tc::tmem_alloc<512>(&tslot);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = tc::idesc_bf16_f32(128, N, 0);
    const uint32_t a0 = tc::smem_u32(sA), b0 = tc::smem_u32(sB);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {                     // K = 128 per iteration
        const uint64_t db = tc::desc_kmajor_sw128(b0 + (kk >> 2) * (N * 128) + (kk & 3) * 32);
        if (TS) {
          tc::mma_bf16_ts(tmem, tmem + 384 + kk * 8, db, idesc, 1u);
        } else {
          const uint64_t da = tc::desc_kmajor_sw128(a0 + (kk >> 2) * 16384 + (kk & 3) * 32);
          tc::mma_bf16_ss(tmem, da, db, idesc, 1u);
        }
      }
      if ((it & 15) == 15) {                               // keep the issue queue bounded
        tc::mma_commit(&bar);
        tc::mbar_wait(&bar, (it >> 4) & 1);
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, (iters >> 4) & 1);
    *sink = tmem;
  }
  tc::tc_fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) { tc::tc_fence_after(); tc::tmem_dealloc<512>(tmem); }
}

template <int N, bool TS>
void run(const char* name, int sms) {
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const int smem = 1024 + 32768 + N * 256;
  cudaFuncSetAttribute(mma_bench<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 20000;
  mma_bench<N, TS><<<sms, 128, smem>>>(100, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  mma_bench<N, TS><<<sms, 128, smem>>>(iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 2.0 * 128 * N * 128 * (double)iters * sms;
  printf("%-28s %8.3f ms  %7.1f TFLOP/s  (%s)\n", name, ms, flops / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<16, false>("M128 N16  SS", sms);
  run<32, false>("M128 N32  SS", sms);
  run<64, false>("M128 N64  SS", sms);
  run<128, false>("M128 N128 SS", sms);
  run<256, false>("M128 N256 SS", sms);
  run<128, true>("M128 N128 TS (A in TMEM)", sms);
  run<256, true>("M128 N256 TS (A in TMEM)", sms);
  return 0;
}
