// k_maint.cu -- cache maintenance: EMA fold, token-selection resolution, payload moves.
//
// The control flow of Alg. 2 -- which sub-cache each token reaches, which
// slot is written, where a selection happens -- depends only on the stream index and
// the counters, never on mu or on the head (the host plan simulates it, plan.cpp).
// What depends on mu is the outcome of each selection.  The device work is:
//
// The EMA fold (P:154 over m rows, Q4) is mu <- g*mu + s in IEEE double (__dmul_rn/__dadd_rn,
// never contracted into an FMA); semantically every fold precedes every insertion (Q9).  Since
// the fold is a pure function of the pre-chunk (mu, s), it is evaluated where it is needed:
//  1. select_resolve: winner of selection k = cand if fold(cand) > fold(inc) else inc
//                (strict '>'), per (b, g), folding both operands on the fly.  Operands
//                that are themselves winners of earlier selections are resolved in
//                dependency-depth order (one launch per depth; depth 0 covers every config).
//  2. maint:     ONE launch: a block per (item, b*g); an item is a range of one phase's slots
//                plus the moves landing in it.  Phases run C_N, ..., C_1, then the sinks.  A
//                block folds the residents of its range in place and writes the range's final
//                occupants (K_raw, V, mu = fold(source), origin).  A slot of C_i only receives
//                tokens from C_{<i} or the chunk, so a block of phase p stores only after every
//                block of phase p-1 is done (device-scope counter per (phase, b*g)) -- those
//                read the slots phase p overwrites -- and its sources are still unfolded,
//                pre-chunk rows, which it loads before waiting.
//
// All HBM-bound: coalesced 16-byte vector copies, a full warp per moved (K | V) row pair.
#include "common.cuh"

namespace cascade {

__device__ __forceinline__ int32_t resolve_ref(int32_t ref, const int32_t* __restrict__ res) {
  return ref >= 0 ? ref : res[-ref - 1];
}

// mu of a concrete source after the fold: g*mu + s of a pre-chunk slot (read unfolded), or s of
// a chunk row (mu starts at 0).
__device__ __forceinline__ double src_mu(const Geometry& g, int32_t x, const double* mu_bg,
                                         const float* s_bg) {
  return x < g.S_tot ? __dadd_rn(__dmul_rn(g.decay, mu_bg[x]), (double)s_bg[x]) : (double)s_bg[x];
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

// One block = one item (a range of <= kMaintSlots slots of one phase, with the <= kMaintMoves
// moves whose destination falls in it) for one (b, g).  Every load (fold operands, source rows)
// is issued before the wait: a block's reads only touch slots of shallower levels and the chunk,
// which no block overwrites before this one publishes.  Only the stores wait for phase p-1.
template <typename T, int VPL>
__global__ void __launch_bounds__(256) maint_kernel(Geometry g, PlanDev p, MaintItems it, StateDev<T> sd,
                                                    const T* __restrict__ k_in, const T* __restrict__ v_in,
                                                    const float* __restrict__ s) {
  __shared__ uint32_t s_ticket;
  if (threadIdx.x == 0) s_ticket = atomicAdd(it.ticket, 1u);
  __syncthreads();
  const int BG = g.B * g.Hkv;
  const uint32_t logical = s_ticket - it.ticket_base;     // start order, not blockIdx: no deadlock
  const int item = (int)(logical / BG), bg = (int)(logical - (uint32_t)item * BG);
  const int4 d = it.items[item];                           // slot_lo, slot_len, move_begin, move_end
  const int phase = it.phase[item];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long sbase = (long long)bg * g.S_tot;
  double* mu = sd.mu + sbase;
  const float* s_bg = s + (long long)bg * (g.S_tot + g.m);

  // fold operands of the slice's pre-chunk residents
  const int lvl = phase < g.N ? g.N - 1 - phase : -1;    // 0-based sub-cache, -1 = sinks
  const int valid_end = min(d.x + d.y, lvl < 0 ? g.sink_pre : g.alpha + lvl * g.c + g.counts_pre[lvl]);
  double f[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int x = d.x + threadIdx.x + j * 256;
    if (x < valid_end) f[j] = __dadd_rn(__dmul_rn(g.decay, mu[x]), (double)s_bg[x]);
  }
  // source rows of the moves: warp w takes moves d.z + w + 8 j; lane l carries 16-byte vectors
  // l, l + 32, ... of the (K | V) row pair
  const int nvec = g.d * (int)sizeof(T) / 16;             // vectors per K (or V) row
  const int gg = bg % g.Hkv, b = bg / g.Hkv;
  const int32_t* res = p.resolved + (long long)bg * p.sel_cap;
  int32_t dst[4];
  int4 buf[4][VPL];
  double mu_new[4];
  int64_t org[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int e = d.z + warp + 8 * j;
    dst[j] = -1;
    if (e < d.w) {
      const int32_t dd = p.mov[2 * e];
      const int32_t src = resolve_ref(p.mov[2 * e + 1], res);
      if (src != dd) {                                     // resident won its selection: stays
        dst[j] = dd;
        const T *ks, *vs;
        if (src < g.S_tot) {
          ks = sd.k_raw + (sbase + src) * g.d;
          vs = sd.v + (sbase + src) * g.d;
          mu_new[j] = __dadd_rn(__dmul_rn(g.decay, mu[src]), (double)s_bg[src]);  // still unfolded
          org[j] = sd.origin[sbase + src];
        } else {
          const int r = src - g.S_tot;
          ks = k_in + (((long long)b * g.m + r) * g.Hkv + gg) * g.d;
          vs = v_in + (((long long)b * g.m + r) * g.Hkv + gg) * g.d;
          mu_new[j] = (double)s_bg[src];
          org[j] = g.t0 + r;
        }
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
          const int i = lane + 32 * u;
          if (i < nvec) buf[j][u] = __ldcs(reinterpret_cast<const int4*>(ks) + i);
          else if (i < 2 * nvec) buf[j][u] = __ldcs(reinterpret_cast<const int4*>(vs) + i - nvec);
        }
      }
    }
  }
  // wait until every block of phase p-1 of this (b, g) is done: they read the slots we overwrite
  if (phase > 0 && phase < g.N) {
    if (threadIdx.x == 0) {
      const uint32_t* ctr = it.done + (phase - 1) * BG + bg;
      const uint32_t want = it.expect[phase - 1];
      uint32_t v;
      while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        if ((int32_t)(v - want) >= 0) break;
        __nanosleep(32);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int x = d.x + threadIdx.x + j * 256;
    if (x < valid_end) mu[x] = f[j];
  }
  __syncthreads();                                         // moves overwrite folded slots' mu
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (dst[j] < 0) continue;
    T* kd = sd.k_raw + (sbase + dst[j]) * g.d;
    T* vd = sd.v + (sbase + dst[j]) * g.d;
#pragma unroll
    for (int u = 0; u < VPL; ++u) {
      const int i = lane + 32 * u;
      if (i < nvec) reinterpret_cast<int4*>(kd)[i] = buf[j][u];
      else if (i < 2 * nvec) reinterpret_cast<int4*>(vd)[i - nvec] = buf[j][u];
    }
    if (lane == 0) {
      mu[dst[j]] = mu_new[j];
      sd.origin[sbase + dst[j]] = org[j];
    }
  }
  // publish completion of this block for the next phase
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(it.done + phase * BG + bg, 1u);
  }
}

template <typename T>
void launch_maint(const Geometry& g, const PlanDev& p, const MaintItems& it, int n_items, StateDev<T> sd,
                  const T* k_in, const T* v_in, const float* s, cudaStream_t st) {
  if (n_items <= 0) return;
  const int vpl = (2 * g.d * (int)sizeof(T) / 16 + 31) / 32;
  const int blocks = n_items * g.B * g.Hkv;
  if (vpl <= 1) maint_kernel<T, 1><<<blocks, 256, 0, st>>>(g, p, it, sd, k_in, v_in, s);
  else maint_kernel<T, 2><<<blocks, 256, 0, st>>>(g, p, it, sd, k_in, v_in, s);
}

template void launch_maint<float>(const Geometry&, const PlanDev&, const MaintItems&, int, StateDev<float>,
                                  const float*, const float*, const float*, cudaStream_t);
template void launch_maint<__nv_bfloat16>(const Geometry&, const PlanDev&, const MaintItems&, int,
                                          StateDev<__nv_bfloat16>, const __nv_bfloat16*, const __nv_bfloat16*,
                                          const float*, cudaStream_t);

__global__ void positions_kernel(Geometry g, int32_t* __restrict__ pe) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < g.S_tot; x += gridDim.x * blockDim.x)
    pe[x] = slot_pe(g, x);
}

void launch_positions(const Geometry& g, int32_t* pe, cudaStream_t st) {
  int blocks = std::min(ceil_div(g.S_tot, 256), 148 * 4);
  positions_kernel<<<blocks, 256, 0, st>>>(g, pe);
}

}  // namespace cascade
