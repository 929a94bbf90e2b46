// Microbenchmark: attainable exp2 rate of pass 2's inner-loop instruction mix (scale FFMA2,
// 12 of 16 exp2 pairs on MUFU + 4 on the FMA pipe, FADD2 accumulate, broadcast float4 bias
// loads from shared memory), values from registers (no TMEM, no MMA), 16 math warps per SM as in
// attn_score_tc.  Reports exp2 per clock per SM against the MUFU-only figure.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o score_mix_bench score_mix_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float2 poly(float2 t) {
  t.x = fmaxf(t.x, -126.f); t.y = fmaxf(t.y, -126.f);
  const float2 j = __fadd2_rn(t, make_float2(12582912.f, 12582912.f));
  const float2 jf = __fadd2_rn(j, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(t, make_float2(-jf.x, -jf.y));
  float2 p = __ffma2_rn(make_float2(0.0551705f, 0.0551705f), f, make_float2(0.2426083f, 0.2426083f));
  p = __ffma2_rn(p, f, make_float2(0.6932609f, 0.6932609f));
  p = __ffma2_rn(p, f, make_float2(0.9999282f, 0.9999282f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(j.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(j.y) << 23)));
}
template <int MODE, int EMU>   // MODE 0: MUFU only; 1: full mix; 2: mix without bias loads
__global__ void __launch_bounds__(512, 1) mix_kernel(float* out, int iters) {
  __shared__ float4 sb[64];
  if (threadIdx.x < 64) sb[threadIdx.x] = make_float4(1.f, 2.f, 3.f, 4.f + threadIdx.x);
  __syncthreads();
  float x[32];
  for (int i = 0; i < 32; ++i) x[i] = -(threadIdx.x & 7) * 0.01f - i * 0.1f;
  float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
  const float2 sc2 = make_float2(0.127f, 0.127f);
  for (int it = 0; it < iters; ++it) {
    const float4* b4 = sb + ((it & 1) * 8);
#pragma unroll
    for (int e = 0; e < 32; e += 4) {
      float4 bb = MODE == 1 ? b4[e >> 2] : make_float4(1.f, 2.f, 3.f, 4.f);
      float2 t0, t1;
      if (MODE == 0) { t0 = make_float2(x[e], x[e + 1]); t1 = make_float2(x[e + 2], x[e + 3]); }
      else {
        t0 = __ffma2_rn(make_float2(x[e], x[e + 1]), sc2, make_float2(-bb.x, -bb.y));
        t1 = __ffma2_rn(make_float2(x[e + 2], x[e + 3]), sc2, make_float2(-bb.z, -bb.w));
      }
      const int q0 = e >> 1, q1 = q0 + 1;
      const bool e0 = MODE != 0 && ((q0 * EMU) % 16) + EMU >= 16, e1 = MODE != 0 && ((q1 * EMU) % 16) + EMU >= 16;
      float2 p0 = e0 ? poly(t0) : make_float2(ex2(t0.x), ex2(t0.y));
      float2 p1 = e1 ? poly(t1) : make_float2(ex2(t1.x), ex2(t1.y));
      if ((e & 4) == 0) { a0 = __fadd2_rn(a0, p0); a1 = __fadd2_rn(a1, p1); }
      else { a2 = __fadd2_rn(a2, p0); a3 = __fadd2_rn(a3, p1); }
    }
    // new operands each round (cheap: one FADD per register would distort; perturb 1 of 32)
    x[0] += 1e-7f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0.x + a0.y + a1.x + a1.y + a2.x + a2.y + a3.x + a3.y;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, sms * 512 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 8192;
  const char* names[] = {"MUFU only (32 ex2 per row-chunk)", "full mix EMU 4/16", "mix EMU 4/16, no bias LDS",
                         "full mix EMU 0/16", "full mix EMU 6/16"};
  for (int k = 0; k < 5; ++k) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (k == 0) mix_kernel<0, 0><<<sms, 512>>>(out, iters);
      if (k == 1) mix_kernel<1, 4><<<sms, 512>>>(out, iters);
      if (k == 2) mix_kernel<2, 4><<<sms, 512>>>(out, iters);
      if (k == 3) mix_kernel<1, 0><<<sms, 512>>>(out, iters);
      if (k == 4) mix_kernel<1, 6><<<sms, 512>>>(out, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double el = (double)sms * 512 * iters * 32;
      if (rep == 2) printf("%-34s %.3f ms  %.2f exp2/clk/SM at %d MHz max clock\n", names[k], ms,
                           el / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
