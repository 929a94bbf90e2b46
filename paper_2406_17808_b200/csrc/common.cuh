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

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace cascade
