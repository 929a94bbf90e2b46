// Microbenchmark: TMEM load / store throughput on this GPU (one CTA per SM), to bound the
// softmax critical path of attention pass 1: per 128-key tile each softmax thread loads its
// row of S (128 fp32 columns) and stores its row of P (64 packed bf16x2 columns).
// Variants: warps per SM (4 = one per SM sub-partition, 8 = two), ld vs st, and loads while
// one thread keeps the tensor pipe busy with M128 N128 K128 MMAs into other TMEM columns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2406_17808_b200/csrc \
//        scripts/micro/tmem_bench.cu -o scripts/micro/tmem_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_util.cuh"
using namespace cascade;

// mode 0: loads (32 columns x 4 per iteration = one 128-column row), 1: stores, 2 / 3: loads /
// stores with concurrent MMAs issued by an extra warp
template <int MODE>
__global__ void tmem_bench(int iters, int ld_warps, unsigned long long* cyc, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); stop = 0; }
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0) tc::tmem_alloc<512>(&tslot);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp < ld_warps) {
    // warp w reaches TMEM lanes 32 (w % 4) .. +31; columns 0..127 (row of S), or 256.. for pair
    const uint32_t base = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128);
    float v[32], acc = 0.f;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (MODE == 1 || MODE == 3) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] = acc + k;
          tc::tmem_st32(base + c * 32, v);
        }
        tc::tmem_wait_st();
        acc += 1.f;
      } else {                                       // the whole row in flight, one wait
        float w[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tc::tmem_ld32(base + c * 32, w[c]);
        tc::tmem_wait_ld();
        float part[16];                              // short independent chains (no FADD latency bound)
#pragma unroll
        for (int k = 0; k < 16; ++k) part[k] = w[0][k] + w[0][k + 16];
#pragma unroll
        for (int c = 1; c < 4; ++c)
#pragma unroll
          for (int k = 0; k < 16; ++k) part[k] += w[c][k] + w[c][k + 16];
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += part[k] * 1e-30f;
      }
    }
    const unsigned long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x * 16 + warp] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (MODE >= 2) {
      __syncwarp();
      if (lane == 0) atomicAdd((int*)&stop, 1);
    }
  } else if (MODE >= 2 && warp == ld_warps && lane == 0) {
    // tensor pipe busy: M128 N128 K128 bf16 MMAs (operands in shared memory) into columns 384..511
    const uint32_t idesc = tc::idesc_bf16_f32(128, 128, 0);
    const uint32_t a0 = tc::smem_u32(smem), b0 = tc::smem_u32(smem + 32768);
    int n = 0;
    const unsigned long long t0 = clock64();
    while (stop < ld_warps) {
#pragma unroll 1
      for (int rep = 0; rep < 4; ++rep)
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t da = tc::desc_kmajor_sw128(a0 + (kk >> 2) * 16384 + (kk & 3) * 32);
        const uint64_t db = tc::desc_kmajor_sw128(b0 + (kk >> 2) * 16384 + (kk & 3) * 32);
        tc::mma_bf16_ss(tmem + 384, da, db, idesc, 1u);
      }
      tc::mma_commit(&bar);
      tc::mbar_wait(&bar, n & 1);
      ++n;
    }
    const unsigned long long t1 = clock64();
    cyc[blockIdx.x * 16 + 15] = (t1 - t0) / (n ? 4 * n : 1);  // clocks per M128 N128 K128 MMA group
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc::tc_fence_after(); tc::tmem_dealloc<512>(tmem); }
}

template <int MODE>
void run(const char* name, int sms, int ld_warps) {
  unsigned long long* cyc;
  float* sink;
  cudaMalloc(&cyc, sms * 16 * 8);
  cudaMemset(cyc, 0, sms * 16 * 8);
  cudaMalloc(&sink, sms * 512 * 4);
  const int smem = 1024 + 65536;
  cudaFuncSetAttribute(tmem_bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int threads = 32 * (ld_warps + (MODE >= 2 ? 1 : 0));
  const int iters = 4096;
  tmem_bench<MODE><<<sms, threads, smem>>>(64, ld_warps, cyc, sink);
  tmem_bench<MODE><<<sms, threads, smem>>>(iters, ld_warps, cyc, sink);
  cudaDeviceSynchronize();
  unsigned long long h[16 * 4];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int w = 0; w < ld_warps; ++w) mean += (double)h[w];
  mean /= ld_warps;
  const double per_row = mean / iters;                 // clocks per 128-column row per warp
  const double bytes_per_clk = (double)ld_warps * 32 * 128 * 4 / per_row;
  printf("%-34s warps %d: %7.1f clk per 128-col row per warp, %6.1f B/clk/SM%s",
         name, ld_warps, per_row, bytes_per_clk, MODE >= 2 ? "" : "\n");
  if (MODE >= 2) printf(", MMA M128N128K128 %llu clk (512 at the nominal peak)\n", h[15]);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("  error: %s\n", cudaGetErrorString(e));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8}) run<0>("tcgen05.ld 32x32b.x32 x4 + wait", sms, w);
  for (int w : {4, 8}) run<1>("tcgen05.st 32x32b.x32 x4 + wait", sms, w);
  for (int w : {4, 8}) run<2>("tcgen05.ld with MMAs running", sms, w);
  for (int w : {4, 8}) run<3>("tcgen05.st with MMAs running", sms, w);
  return 0;
}
