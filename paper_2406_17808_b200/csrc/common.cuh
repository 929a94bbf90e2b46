// common.cuh -- device helpers shared by the kernels (library-private).
#pragma once

#include <algorithm>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "internal.h"

namespace cascade {

template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Iterate over the valid pre-chunk resident runs: sinks, then sub-caches 1..N (slot order).
// Returns the number of runs; run j covers flat slots [beg[j], beg[j] + len[j]).
__device__ __forceinline__ int resident_runs(const Geometry& g, int32_t* beg, int32_t* len) {
  int n = 0;
  beg[n] = 0; len[n] = g.sink_pre; ++n;
  for (int i = 0; i < g.N; ++i) { beg[n] = g.alpha + i * g.c; len[n] = g.counts_pre[i]; ++n; }
  return n;
}

// Head-reduction ablations of s_g over the group's per-head masses v[0..G):
// 1 = mean (summed in head order), 2 = median (even G: the mean of the two middle values, as
// numpy's median).  Sorts v in place.  The default reduction, max, stays inline at each call site.
constexpr int kMaxMedianGroup = 32;
__device__ inline float group_reduce_ablation(float* v, int G, int mode) {
  if (mode == 1) {
    float sum = 0.f;
    for (int i = 0; i < G; ++i) sum += v[i];
    return __fdiv_rn(sum, (float)G);
  }
  for (int i = 1; i < G; ++i) {                    // insertion sort, G <= kMaxMedianGroup
    const float x = v[i];
    int j = i - 1;
    while (j >= 0 && v[j] > x) { v[j + 1] = v[j]; --j; }
    v[j + 1] = x;
  }
  return (G & 1) ? v[G / 2] : __fdiv_rn(v[G / 2 - 1] + v[G / 2], 2.f);
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace cascade
