// k_maint.cu -- cache maintenance: EMA fold, token-selection resolution, payload moves.
//
// The control flow of Alg. 2 -- which sub-cache each token reaches, which
// slot is written, where a selection happens -- depends only on the stream index and
// the counters, never on mu or on the head (the host plan simulates it, plan.cpp).
// What depends on mu is the outcome of each selection.  The device work is:
//
//  1. ema_fold:  mu <- g*mu + s for every pre-chunk resident (P:154 over m rows, Q4),
//                IEEE double, __dmul_rn/__dadd_rn so nothing is contracted into an FMA.
//                All folds precede all insertions (Q9).
//  2. select_resolve: winner of selection k = cand if mu(cand) > mu(inc) else inc
//                (strict '>'), per (b, g).  Operands that are themselves winners
//                of earlier selections are resolved in dependency-depth order (one
//                launch per depth; depth 0 covers every config in BASELINE.json).
//  3. moves:     per sub-cache, from C_N down to C_1 then the sinks, copy the final
//                occupant of every written slot (K_raw, V, mu, origin).  A slot of
//                C_i only ever receives tokens from C_{<i} or the chunk, so writing
//                the deepest sub-cache first never overwrites a source still to be read.
//
// All HBM-bound: coalesced 16-byte vector copies, one warp per (row, head).
#include "common.cuh"

namespace cascade {

__global__ void ema_fold_kernel(Geometry g, double* __restrict__ mu, const float* __restrict__ s) {
  const long long total = (long long)g.B * g.Hkv * g.S_tot;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % g.S_tot);
    const long long bg = i / g.S_tot;
    if (slot_pe(g, x) < 0) continue;
    const double sv = (double)s[bg * (g.S_tot + g.m) + x];
    mu[i] = __dadd_rn(__dmul_rn(g.decay, mu[i]), sv);
  }
}

void launch_ema_fold(const Geometry& g, double* mu, const float* s, cudaStream_t st) {
  long long total = (long long)g.B * g.Hkv * g.S_tot;
  int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  ema_fold_kernel<<<blocks, 256, 0, st>>>(g, mu, s);
}

__device__ __forceinline__ int32_t resolve_ref(int32_t ref, const int32_t* __restrict__ res) {
  return ref >= 0 ? ref : res[-ref - 1];
}

// mu of a concrete source: folded mu of a pre-chunk slot, or s of a chunk row (mu starts at 0).
__device__ __forceinline__ double src_mu(const Geometry& g, int32_t x, const double* mu_bg,
                                         const float* s_bg) {
  return x < g.S_tot ? mu_bg[x] : (double)s_bg[x];
}

__global__ void select_resolve_kernel(Geometry g, PlanDev p, int32_t begin, int32_t end,
                                      const double* __restrict__ mu, const float* __restrict__ s) {
  const int n = end - begin;
  const long long total = (long long)n * g.B * g.Hkv;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long bg = i / n;
    const int j = begin + (int)(i - bg * n);
    const int k = p.sel_order[j];
    int32_t* res = p.resolved + bg * p.sel_cap;
    const int32_t cand = resolve_ref(p.sel[3 * k + 1], res);
    const int32_t inc = resolve_ref(p.sel[3 * k + 2], res);
    const double* mu_bg = mu + bg * g.S_tot;
    const float* s_bg = s + bg * (g.S_tot + g.m);
    res[k] = src_mu(g, cand, mu_bg, s_bg) > src_mu(g, inc, mu_bg, s_bg) ? cand : inc;
  }
}

void launch_select_resolve(const Geometry& g, const PlanDev& p, int32_t begin, int32_t end,
                           const double* mu, const float* s, cudaStream_t st) {
  long long total = (long long)(end - begin) * g.B * g.Hkv;
  if (total <= 0) return;
  int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  select_resolve_kernel<<<blocks, 256, 0, st>>>(g, p, begin, end, mu, s);
}

// One warp per (move entry, b, g): row copy with 16-byte vectors.
template <typename T>
__global__ void moves_kernel(Geometry g, PlanDev p, int32_t begin, int32_t end, StateDev<T> sd,
                             const T* __restrict__ k_in, const T* __restrict__ v_in,
                             const float* __restrict__ s) {
  const int lane = threadIdx.x & 31;
  const int n = end - begin;
  const long long total = (long long)n * g.B * g.Hkv;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; w < total; w += nwarps) {
    const long long bg = w / n;
    const int e = begin + (int)(w - bg * n);
    const int32_t dst = p.mov[2 * e];
    const int32_t src = resolve_ref(p.mov[2 * e + 1], p.resolved + bg * p.sel_cap);
    if (src == dst) continue;                      // resident won its selection: already in place
    const int gg = (int)(bg % g.Hkv), b = (int)(bg / g.Hkv);
    const T *ks, *vs;
    double mu_new;
    int64_t org;
    if (src < g.S_tot) {
      ks = sd.k_raw + (bg * g.S_tot + src) * g.d;
      vs = sd.v + (bg * g.S_tot + src) * g.d;
      mu_new = sd.mu[bg * g.S_tot + src];
      org = sd.origin[bg * g.S_tot + src];
    } else {
      const int r = src - g.S_tot;
      ks = k_in + (((long long)b * g.m + r) * g.Hkv + gg) * g.d;
      vs = v_in + (((long long)b * g.m + r) * g.Hkv + gg) * g.d;
      mu_new = (double)s[bg * (g.S_tot + g.m) + src];
      org = g.t0 + r;
    }
    T* kd = sd.k_raw + (bg * g.S_tot + dst) * g.d;
    T* vd = sd.v + (bg * g.S_tot + dst) * g.d;
    const int nvec = g.d * (int)sizeof(T) / 16;    // 16-byte vectors per row
    for (int i = lane; i < nvec; i += 32) {
      reinterpret_cast<int4*>(kd)[i] = reinterpret_cast<const int4*>(ks)[i];
      reinterpret_cast<int4*>(vd)[i] = reinterpret_cast<const int4*>(vs)[i];
    }
    if (lane == 0) {
      sd.mu[bg * g.S_tot + dst] = mu_new;
      sd.origin[bg * g.S_tot + dst] = org;
    }
  }
}

template <typename T>
void launch_moves(const Geometry& g, const PlanDev& p, int32_t begin, int32_t end, StateDev<T> sd,
                  const T* k_in, const T* v_in, const float* s, cudaStream_t st) {
  long long total = (long long)(end - begin) * g.B * g.Hkv;
  if (total <= 0) return;
  int blocks = (int)std::min<long long>((total * 32 + 255) / 256, 148LL * 16);
  moves_kernel<T><<<blocks, 256, 0, st>>>(g, p, begin, end, sd, k_in, v_in, s);
}

template void launch_moves<float>(const Geometry&, const PlanDev&, int32_t, int32_t, StateDev<float>,
                                  const float*, const float*, const float*, cudaStream_t);
template void launch_moves<__nv_bfloat16>(const Geometry&, const PlanDev&, int32_t, int32_t,
                                          StateDev<__nv_bfloat16>, const __nv_bfloat16*,
                                          const __nv_bfloat16*, const float*, cudaStream_t);

__global__ void positions_kernel(Geometry g, int32_t* __restrict__ pe) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < g.S_tot; x += gridDim.x * blockDim.x)
    pe[x] = slot_pe(g, x);
}

void launch_positions(const Geometry& g, int32_t* pe, cudaStream_t st) {
  int blocks = std::min(ceil_div(g.S_tot, 256), 148 * 4);
  positions_kernel<<<blocks, 256, 0, st>>>(g, pe);
}

}  // namespace cascade
