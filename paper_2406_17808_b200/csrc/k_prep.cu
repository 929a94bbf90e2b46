// k_prep.cu -- RoPE by cache rank + layout prep for the attention passes.
//
// Writes, for one layer and one chunk:
//   q_rot  [B][Hq][ldc][d]          chunk queries rotated to pe = n_cached + r
//   k_rot  [B][Hkv][S_tot + ldc][d] resident keys (flat slot order) rotated to their pre-chunk
//                                   rank pe (closed form, slot_pe), chunk keys at rows S_tot + r
//                                   rotated to n_cached + r
//   v_chunk[B][Hkv][ldc][d]         chunk values, head-major
// Keys are cached pre-RoPE (Q11) because ranks change every chunk.  cos/sin come from a table
// built on the host in float64 (rope_tab[pos][i], and its float rounding rope_tab_f); the
// rotated bf16 operand is the float64 rotation's rounding (Q17), see rotate().
//
// HBM-bound: every thread moves one 16-byte vector of the first half of a row and the
// matching vector of the second half (rotate-half pairs (i, i + d/2)), so D/(2*EPV) threads
// cover a row (8 for bf16 d = 128) with fully coalesced 16-byte loads and stores.
#include "common.cuh"

#include <type_traits>

namespace cascade {

namespace {

template <typename T> struct Vec;
template <> struct Vec<float> {
  static constexpr int N = 4;
  __device__ static void unpack(const uint4& u, float* f) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y); f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  }
  __device__ static uint4 pack(const float* f) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
  }
};
template <> struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ static void unpack(const uint4& u, float* f) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
  __device__ static uint4 pack(const float* f) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
      w[i] = *reinterpret_cast<const uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};

// rotate-half on one vector pair: lo = x[i..i+N), hi = x[i+d/2 .. i+d/2+N) at frequencies i..i+N.
// The reference result (reading Q17) is the oracle's: the rotation in double with separately
// rounded products (never an FMA), rounded double -> float -> T.  Computing it in double for every
// element costs DMUL/DADD issue and a 16-byte table entry per element (cfg3: 54 vs 26 ms per
// step), so the bf16 path rotates in float first and keeps that result only when it PROVABLY
// rounds to the same bf16:  with c, s the float roundings of the double table (|err| <= 2^-24)
// and y = fma(x1, c, -(x2 s)),  |y - Y| <= 2^-23 (|x1| + |x2|) + 2^-24 |y|  for the exact
// Y = x1 C - x2 S, and the double result and its float rounding lie within another 2^-24 |Y|.
// E = 2^-22 (|x1| + |x2| + |y|) covers all of it; if no bf16 rounding midpoint lies within E of
// y, every value of [y - E, y + E] -- y and the reference among them -- rounds to the same bf16.
// Otherwise (about 1e-4 of the elements) the element is recomputed the reference way.  fp32 (the
// toy path) keeps the float output of the double rotation.
__device__ __forceinline__ bool bf16_round_safe(float y, float E) {
  const uint32_t u = __float_as_uint(y);
  const int dm = abs((int)(u & 0xFFFFu) - 0x8000);          // float ulps to the nearest midpoint
  const float ulp = __uint_as_float(u & 0x7F800000u) * 1.1920928955078125e-7f;   // 2^(e-150)
  return (float)dm * ulp > E;                               // 0 / subnormal y: ulp 0 -> false
}

template <typename T>
__device__ __forceinline__ void rotate(uint4& lo, uint4& hi, const double2* __restrict__ cs,
                                       const float2* __restrict__ csf) {
  constexpr int N = Vec<T>::N;
  float a[N], b[N];
  Vec<T>::unpack(lo, a);
  Vec<T>::unpack(hi, b);
#pragma unroll
  for (int e = 0; e < N; ++e) {
    const float x1 = a[e], x2 = b[e];
    bool exact = !std::is_same<T, __nv_bfloat16>::value;
    if (!exact) {
      const float2 c = csf[e];
      const float ya = fmaf(x1, c.x, -(x2 * c.y));
      const float yb = fmaf(x2, c.x, x1 * c.y);
      const float sx = fabsf(x1) + fabsf(x2);
      exact = !(bf16_round_safe(ya, (sx + fabsf(ya)) * 2.384185791015625e-7f) &&
                bf16_round_safe(yb, (sx + fabsf(yb)) * 2.384185791015625e-7f));    // 2^-22
      a[e] = ya;
      b[e] = yb;
    }
    if (exact) {
      const double2 c = cs[e];
      a[e] = __double2float_rn(__dsub_rn(__dmul_rn((double)x1, c.x), __dmul_rn((double)x2, c.y)));
      b[e] = __double2float_rn(__dadd_rn(__dmul_rn((double)x2, c.x), __dmul_rn((double)x1, c.y)));
    }
  }
  lo = Vec<T>::pack(a);
  hi = Vec<T>::pack(b);
}

}  // namespace

// I: index type of the task / row arithmetic -- 32-bit whenever the task count fits (the
// divisions by Hq, S_tot + m, Hkv and m are then 32-bit, a fraction of the 64-bit cost)
template <typename T, typename I>
__global__ void __launch_bounds__(256) rope_prep_kernel(Geometry g, const T* __restrict__ q, const T* __restrict__ k,
                                                        const T* __restrict__ v, const T* __restrict__ k_raw,
                                                        const double2* __restrict__ tab,
                                                        const float2* __restrict__ tabf, T* __restrict__ q_rot,
                                                        T* __restrict__ k_rot, T* __restrict__ v_chunk) {
  constexpr int N = Vec<T>::N;                 // elements per 16-byte vector
  const int half = g.d >> 1;
  const int tpr = half / N;                    // threads per row (a power of two)
  const int tpr_log2 = __ffs(tpr) - 1;
  const I rows_q = (I)g.B * g.m * g.Hq;
  const I rows_k = (I)g.B * g.Hkv * (g.S_tot + g.m);
  const I rows_v = (I)g.B * g.m * g.Hkv;
  const I total = (rows_q + rows_k + rows_v) * tpr;
  for (I task = blockIdx.x * (I)blockDim.x + threadIdx.x; task < total; task += (I)gridDim.x * blockDim.x) {
    I row = task >> tpr_log2;
    const int t = (int)(task & (tpr - 1));
    const int i0 = t * N;                      // first frequency index of this thread
    if (row < rows_q) {                        // source order (b, r, h): contiguous reads
      const int h = (int)(row % (I)g.Hq);
      const I br = row / (I)g.Hq;
      const int r = (int)(br % (I)g.m), b = (int)(br / (I)g.m);
      const uint4* src = reinterpret_cast<const uint4*>(q + (long long)row * g.d);
      uint4 lo = src[t], hi = src[t + tpr];
      rotate<T>(lo, hi, tab + (long long)(g.n_cached + r) * half + i0, tabf + (long long)(g.n_cached + r) * half + i0);
      uint4* dst = reinterpret_cast<uint4*>(q_rot + (((long long)b * g.Hq + h) * g.ldc + r) * g.d);
      dst[t] = lo; dst[t + tpr] = hi;
      continue;
    }
    row -= rows_q;
    if (row < rows_k) {
      const I ld = (I)(g.S_tot + g.m);
      const int x = (int)(row % ld);
      const long long bg = (long long)(row / ld);
      const uint4* src;
      int pe;
      if (x < g.S_tot) {
        pe = slot_pe(g, x);
        if (pe < 0) continue;                  // empty slot: never read
        src = reinterpret_cast<const uint4*>(k_raw + (bg * g.S_tot + x) * g.d);
      } else {
        const int r = x - g.S_tot;
        const int gg = (int)(bg % g.Hkv), b = (int)(bg / g.Hkv);
        pe = g.n_cached + r;
        src = reinterpret_cast<const uint4*>(k + (((long long)b * g.m + r) * g.Hkv + gg) * g.d);
      }
      uint4 lo = src[t], hi = src[t + tpr];
      rotate<T>(lo, hi, tab + (long long)pe * half + i0, tabf + (long long)pe * half + i0);
      uint4* dst = reinterpret_cast<uint4*>(k_rot + (bg * (g.S_tot + g.ldc) + x) * g.d);
      dst[t] = lo; dst[t + tpr] = hi;
      continue;
    }
    row -= rows_k;                             // v_chunk[b][g][r] <- v[b][r][g]
    {
      const int gg = (int)(row % (I)g.Hkv);
      const I br = row / (I)g.Hkv;
      const int r = (int)(br % (I)g.m), b = (int)(br / (I)g.m);
      const uint4* src = reinterpret_cast<const uint4*>(v + (long long)row * g.d);
      uint4* dst = reinterpret_cast<uint4*>(v_chunk + (((long long)b * g.Hkv + gg) * g.ldc + r) * g.d);
      dst[t] = src[t]; dst[t + tpr] = src[t + tpr];
    }
  }
}

template <typename T>
void launch_rope_prep(const Geometry& g, const T* q, const T* k, const T* v, const T* k_raw_state,
                      const double2* rope_tab, const float2* rope_tab_f, T* q_rot, T* k_rot, T* v_chunk,
                      cudaStream_t st) {
  const int tpr = (g.d / 2) / Vec<T>::N;
  const long long total = ((long long)g.B * g.Hq * g.m + (long long)g.B * g.Hkv * (g.S_tot + g.m) +
                           (long long)g.B * g.Hkv * g.m) * tpr;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 8);
  if (total + 148LL * 8 * 256 < (1LL << 31))
    rope_prep_kernel<T, uint32_t><<<blocks, 256, 0, st>>>(g, q, k, v, k_raw_state, rope_tab, rope_tab_f, q_rot, k_rot, v_chunk);
  else
    rope_prep_kernel<T, long long><<<blocks, 256, 0, st>>>(g, q, k, v, k_raw_state, rope_tab, rope_tab_f, q_rot, k_rot, v_chunk);
}

template void launch_rope_prep<float>(const Geometry&, const float*, const float*, const float*,
                                      const float*, const double2*, const float2*, float*, float*, float*,
                                      cudaStream_t);
template void launch_rope_prep<__nv_bfloat16>(const Geometry&, const __nv_bfloat16*, const __nv_bfloat16*,
                                              const __nv_bfloat16*, const __nv_bfloat16*, const double2*,
                                              const float2*, __nv_bfloat16*, __nv_bfloat16*, __nv_bfloat16*,
                                              cudaStream_t);

}  // namespace cascade
