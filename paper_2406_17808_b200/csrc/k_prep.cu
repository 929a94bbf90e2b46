// k_prep.cu -- RoPE by cache rank + layout prep for the attention passes.
//
// Writes, for one layer and one chunk:
//   q_rot  [B][Hq][ldc][d]        chunk queries rotated to pe = n_cached + r
//   k_rot  [B][Hkv][S_tot + ldc][d] resident keys (flat slot order) rotated to their
//                                 pre-chunk rank pe (closed form, slot_pe), and chunk
//                                 keys at rows S_tot + r rotated to n_cached + r
//   v_chunk[B][Hkv][ldc][d]       chunk values, head-major
// Keys are cached pre-RoPE (Q11) because ranks change every chunk.  cos/sin come
// from a table built on the host in float64 and rounded to fp32 (rope_tab[pos][i]).
// HBM-bound elementwise work: one thread per rotate-half pair, coalesced along d.
#include "common.cuh"

namespace cascade {

template <typename T>
__global__ void rope_prep_kernel(Geometry g, const T* __restrict__ q, const T* __restrict__ k,
                                 const T* __restrict__ v, const T* __restrict__ k_raw,
                                 const float2* __restrict__ tab, T* __restrict__ q_rot,
                                 T* __restrict__ k_rot, T* __restrict__ v_chunk) {
  const int half = g.d >> 1;
  const long long rows_q = (long long)g.B * g.Hq * g.m;
  const long long rows_k = (long long)g.B * g.Hkv * (g.S_tot + g.m);
  const long long rows_v = (long long)g.B * g.Hkv * g.m;
  const long long total = (rows_q + rows_k + rows_v) * half;
  for (long long task = blockIdx.x * (long long)blockDim.x + threadIdx.x; task < total;
       task += (long long)gridDim.x * blockDim.x) {
    long long row = task / half;
    int i = (int)(task - row * half);
    if (row < rows_q) {                       // q_rot[b][h][r] <- rope(q[b][r][h], n_c + r)
      int r = (int)(row % g.m);
      long long bh = row / g.m;
      int h = (int)(bh % g.Hq), b = (int)(bh / g.Hq);
      const T* src = q + (((long long)b * g.m + r) * g.Hq + h) * g.d;
      float2 cs = tab[(long long)(g.n_cached + r) * half + i];
      float x1 = to_f(src[i]), x2 = to_f(src[i + half]);
      T* dst = q_rot + (bh * g.ldc + r) * g.d;
      dst[i] = from_f<T>(x1 * cs.x - x2 * cs.y);
      dst[i + half] = from_f<T>(x2 * cs.x + x1 * cs.y);
      continue;
    }
    row -= rows_q;
    if (row < rows_k) {
      const int ld = g.S_tot + g.m;
      int x = (int)(row % ld);
      long long bg = row / ld;
      const T* src;
      int pe;
      if (x < g.S_tot) {
        pe = slot_pe(g, x);
        if (pe < 0) continue;                 // empty slot: never read
        src = k_raw + (bg * g.S_tot + x) * g.d;
      } else {
        int r = x - g.S_tot;
        int gg = (int)(bg % g.Hkv), b = (int)(bg / g.Hkv);
        pe = g.n_cached + r;
        src = k + (((long long)b * g.m + r) * g.Hkv + gg) * g.d;
      }
      float2 cs = tab[(long long)pe * half + i];
      float x1 = to_f(src[i]), x2 = to_f(src[i + half]);
      T* dst = k_rot + (bg * (g.S_tot + g.ldc) + x) * g.d;
      dst[i] = from_f<T>(x1 * cs.x - x2 * cs.y);
      dst[i + half] = from_f<T>(x2 * cs.x + x1 * cs.y);
      continue;
    }
    row -= rows_k;                            // v_chunk[b][g][r] <- v[b][r][g]
    {
      int r = (int)(row % g.m);
      long long bg = row / g.m;
      int gg = (int)(bg % g.Hkv), b = (int)(bg / g.Hkv);
      const T* src = v + (((long long)b * g.m + r) * g.Hkv + gg) * g.d;
      T* dst = v_chunk + (bg * g.ldc + r) * g.d;
      dst[i] = src[i];
      dst[i + half] = src[i + half];
    }
  }
}

template <typename T>
void launch_rope_prep(const Geometry& g, const T* q, const T* k, const T* v, const T* k_raw_state,
                      const float2* rope_tab, T* q_rot, T* k_rot, T* v_chunk, cudaStream_t st) {
  long long total = ((long long)g.B * g.Hq * g.m + (long long)g.B * g.Hkv * (g.S_tot + g.m) +
                     (long long)g.B * g.Hkv * g.m) * (g.d / 2);
  int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  rope_prep_kernel<T><<<blocks, 256, 0, st>>>(g, q, k, v, k_raw_state, rope_tab, q_rot, k_rot, v_chunk);
}

template void launch_rope_prep<float>(const Geometry&, const float*, const float*, const float*,
                                      const float*, const float2*, float*, float*, float*, cudaStream_t);
template void launch_rope_prep<__nv_bfloat16>(const Geometry&, const __nv_bfloat16*, const __nv_bfloat16*,
                                              const __nv_bfloat16*, const __nv_bfloat16*, const float2*,
                                              __nv_bfloat16*, __nv_bfloat16*, __nv_bfloat16*, cudaStream_t);

}  // namespace cascade
