// k_attn_simt.cu -- exact SIMT (FFMA) attention + per-key EMA mass.
//
// This is the fp32 path (cfg1 toy, BASELINE configs[0]): tf32 tensor cores cannot meet
// the 1e-4 max-abs bar, so fp32 runs on the FFMA pipe with expf.  It also serves as
// the bring-up path for bf16 until the tcgen05 kernels take over.
//
// Pass 1 (attn_fwd_simt): one warp per (b, h, r).  The query attends to every valid
//   resident slot and to chunk keys r' <= r (Fig. 4 slice) with an online
//   softmax; writes O[b][r][h] and the row log-sum-exp (natural log).
// Pass 2 (attn_score_simt): one warp per (b, g, key).  Recomputes the logits with the
//   final LSE so the probabilities are exact (reading Q6), accumulates
//   s_h = sum_r w_r P_h[r, key] with w_r = (1 - gamma) gamma^(m-1-r) (Alg. 3 C_EMA,
//   P:644), and writes s_g = max over the G q-heads of the group.
#include "common.cuh"

namespace cascade {

template <typename T, int D>
__global__ void attn_fwd_simt_kernel(Geometry g, const T* __restrict__ q_rot,
                                     const T* __restrict__ k_rot, const T* __restrict__ v_state,
                                     const T* __restrict__ v_chunk, T* __restrict__ out,
                                     float* __restrict__ lse) {
  constexpr int E = D / 32;
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nrows = (long long)g.B * g.Hq * g.m;
  if (warp >= nrows) return;
  const int r = (int)(warp % g.m);
  const int h = (int)((warp / g.m) % g.Hq);
  const int b = (int)(warp / ((long long)g.m * g.Hq));
  const int gg = h / g.G;
  const long long bg = (long long)b * g.Hkv + gg;

  float qv[E], o[E];
  const T* qp = q_rot + (((long long)b * g.Hq + h) * g.ldc + r) * D;
#pragma unroll
  for (int e = 0; e < E; ++e) { qv[e] = to_f(qp[lane + 32 * e]); o[e] = 0.f; }
  float mrun = -INFINITY, l = 0.f;

  const T* kbase = k_rot + bg * (long long)(g.S_tot + g.ldc) * D;
  auto visit = [&](const T* kp, const T* vp) {
    float part = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) part += qv[e] * to_f(kp[lane + 32 * e]);
    float logit = warp_sum(part) * g.scale;
    float mnew = fmaxf(mrun, logit);
    float corr = expf(mrun - mnew);
    float p = expf(logit - mnew);
    l = l * corr + p;
#pragma unroll
    for (int e = 0; e < E; ++e) o[e] = o[e] * corr + p * to_f(vp[lane + 32 * e]);
    mrun = mnew;
  };

  int32_t beg[CASCADE_MAX_LEVELS + 1], len[CASCADE_MAX_LEVELS + 1];
  int nr = resident_runs(g, beg, len);
  for (int j = 0; j < nr; ++j)
    for (int x = beg[j]; x < beg[j] + len[j]; ++x)
      visit(kbase + (long long)x * D, v_state + (bg * g.S_tot + x) * D);
  for (int rr = 0; rr <= r; ++rr)
    visit(kbase + (long long)(g.S_tot + rr) * D, v_chunk + (bg * g.ldc + rr) * D);

  const float inv = 1.f / l;
  T* op = out + (((long long)b * g.m + r) * g.Hq + h) * D;
#pragma unroll
  for (int e = 0; e < E; ++e) op[lane + 32 * e] = from_f<T>(o[e] * inv);
  if (lane == 0) lse[((long long)b * g.Hq + h) * g.ldc + r] = mrun + logf(l);
}

template <typename T, int D>
__global__ void attn_score_simt_kernel(Geometry g, const T* __restrict__ q_rot,
                                       const T* __restrict__ k_rot, const float* __restrict__ lse,
                                       const float* __restrict__ w, float* __restrict__ s,
                                       float* __restrict__ heads_out, int heads_ld) {
  constexpr int E = D / 32;
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int ld = g.S_tot + g.m;
  const long long nkeys = (long long)g.B * g.Hkv * ld;
  if (warp >= nkeys) return;
  const int x = (int)(warp % ld);
  const long long bg = warp / ld;
  const int gg = (int)(bg % g.Hkv), b = (int)(bg / g.Hkv);

  int r_lo;
  if (x < g.S_tot) {
    if (slot_pe(g, x) < 0) { if (lane == 0) s[warp] = 0.f; return; }
    r_lo = 0;
  } else {
    r_lo = x - g.S_tot;
  }
  float kv[E];
  const T* kp = k_rot + (bg * (g.S_tot + g.ldc) + x) * D;
#pragma unroll
  for (int e = 0; e < E; ++e) kv[e] = to_f(kp[lane + 32 * e]);

  float best = 0.f;
  float hv[kMaxMedianGroup];
  for (int j = 0; j < g.G; ++j) {
    const int h = gg * g.G + j;
    const T* qb = q_rot + ((long long)b * g.Hq + h) * g.ldc * D;
    const float* lb = lse + ((long long)b * g.Hq + h) * g.ldc;
    float acc = 0.f;
    for (int r = r_lo; r < g.m; ++r) {
      float part = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) part += kv[e] * to_f(qb[(long long)r * D + lane + 32 * e]);
      float logit = warp_sum(part) * g.scale;
      acc += w[r] * expf(logit - lb[r]);
    }
    best = j == 0 ? acc : fmaxf(best, acc);       // max over the group
    if (j < kMaxMedianGroup) hv[j] = acc;         // G <= 32 whenever an ablation is on
    if (heads_out && lane == 0) heads_out[((long long)b * g.Hq + h) * heads_ld + x] = acc;
  }
  if (g.head_reduce) best = group_reduce_ablation(hv, g.G, g.head_reduce);   // mean / median
  if (lane == 0) s[warp] = best;
}

template <typename T>
void launch_attn_fwd_simt(const Geometry& g, const T* q_rot, const T* k_rot, const T* v_state,
                          const T* v_chunk, T* out, float* lse, cudaStream_t st) {
  long long warps = (long long)g.B * g.Hq * g.m;
  int blocks = ceil_div(warps * 32, 256);
  if (g.d == 64)
    attn_fwd_simt_kernel<T, 64><<<blocks, 256, 0, st>>>(g, q_rot, k_rot, v_state, v_chunk, out, lse);
  else
    attn_fwd_simt_kernel<T, 128><<<blocks, 256, 0, st>>>(g, q_rot, k_rot, v_state, v_chunk, out, lse);
}

template <typename T>
void launch_attn_score_simt(const Geometry& g, const T* q_rot, const T* k_rot, const float* lse,
                            const float* w, float* s, float* heads_out, int heads_ld, cudaStream_t st) {
  long long warps = (long long)g.B * g.Hkv * (g.S_tot + g.m);
  int blocks = ceil_div(warps * 32, 256);
  if (g.d == 64)
    attn_score_simt_kernel<T, 64><<<blocks, 256, 0, st>>>(g, q_rot, k_rot, lse, w, s, heads_out, heads_ld);
  else
    attn_score_simt_kernel<T, 128><<<blocks, 256, 0, st>>>(g, q_rot, k_rot, lse, w, s, heads_out, heads_ld);
}

#define INST(T)                                                                                   \
  template void launch_attn_fwd_simt<T>(const Geometry&, const T*, const T*, const T*, const T*, \
                                        T*, float*, cudaStream_t);                              \
  template void launch_attn_score_simt<T>(const Geometry&, const T*, const T*, const float*,     \
                                          const float*, float*, float*, int, cudaStream_t);
INST(float)   // the fp32 path only: bf16 runs the tcgen05 kernels (k_attn_tc.cu)
#undef INST

}  // namespace cascade
