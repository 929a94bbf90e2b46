// k_maint.cu -- cache maintenance: EMA fold, token-selection resolution, payload moves.
//
// The control flow of Alg. 2 -- which sub-cache each token reaches, which
// slot is written, where a selection happens -- depends only on the stream index and
// the counters, never on mu or on the head (the host plan simulates it, plan.cpp).
// What depends on mu is the outcome of each selection.  The device work is:
//
//  0. EMA fold (P:154 over m rows, Q4): mu <- g*mu + s in IEEE double (__dmul_rn/__dadd_rn,
//     never contracted into an FMA), before any insertion (Q9).  The tcgen05 pass 2 does it in
//     its epilogue; ema_fold_kernel serves score injection and the SIMT path.
//  1. select_resolve (only when a selection operand is itself a selection of the same chunk,
//     i.e. m > c wraps a level): winner = cand if mu(cand) > mu(inc) else inc (strict '>',
//     P:615), per (b, g), one launch per dependency depth.  Depth-0 selections -- all of them
//     in every benchmark config -- are resolved inside the block that moves the winner.
//  2. maint: ONE launch, a block per (item, b*g).  An item is a run of <= 64 moves of one
//     phase (phases C_N, ..., C_1, sinks; destinations sorted), with at most kMaintStaged
//     moves that read a resident slot.  Hazard: a move's source may be a pre-chunk slot that
//     another item overwrites (an evictee carried to the next sub-cache).  The host
//     lists, per item, the items that READ its destinations (always earlier items, deeper
//     sub-caches); a block loads resident sources into shared memory (cp.async), publishes
//     "loaded" (a per-(item, b*g) epoch flag), waits only for the flags of its readers, then
//     stores.  Chunk-row sources are never overwritten: copied after the wait, straight
//     through registers.
//
// All HBM-bound: coalesced 16-byte vectors, a full warp per moved (K | V) row pair.
#include "common.cuh"

namespace cascade {

__device__ __forceinline__ uint32_t tc_smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ int32_t resolve_ref(int32_t ref, const int32_t* __restrict__ res) {
  return ref >= 0 ? ref : res[-ref - 1];
}

// mu of a concrete source after the fold: the folded mu of a pre-chunk slot, or s of a chunk
// row (mu starts at 0).
__device__ __forceinline__ double src_mu(const Geometry& g, int32_t x, const double* mu_bg,
                                         const float* s_bg) {
  return x < g.S_tot ? mu_bg[x] : (double)s_bg[x];
}

__global__ void ema_fold_kernel(Geometry g, double* __restrict__ mu, const float* __restrict__ s) {
  const int BG = g.B * g.Hkv;
  const long long total = (long long)BG * g.S_tot;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long bg = i / g.S_tot;
    const int x = (int)(i - bg * g.S_tot);
    bool valid = x < g.sink_pre;
    if (x >= g.alpha) {
      const int lvl = (x - g.alpha) / g.c;
      int cnt = 0;
#pragma unroll
      for (int k = 0; k < CASCADE_MAX_LEVELS; ++k) cnt = k == lvl ? g.counts_pre[k] : cnt;
      valid = x - g.alpha - lvl * g.c < cnt;
    }
    if (valid) mu[i] = __dadd_rn(__dmul_rn(g.decay, mu[i]), (double)s[bg * (g.S_tot + g.m) + x]);
  }
}

void launch_ema_fold(const Geometry& g, double* mu, const float* s, cudaStream_t st) {
  const long long total = (long long)g.B * g.Hkv * g.S_tot;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 8);
  ema_fold_kernel<<<blocks, 256, 0, st>>>(g, mu, s);
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

// maint_kernel: one block (8 warps) = one item for one (b, g).  Warp w owns moves 8w .. 8w+7 of
// the item; lane j < 8 resolves move j (source, destination, mu, origin stay in its registers).
// Every move of an item reads a resident slot; all rows go to shared memory before publishing.
template <typename T>
__global__ void __launch_bounds__(256, 6) maint_kernel(Geometry g, PlanDev p, MaintItems it, StateDev<T> sd,
                                                       const float* __restrict__ s) {
  constexpr int kPerWarp = kMaintMoves / 8;
  extern __shared__ __align__(16) int4 s_rows[];          // [kMaintMoves][2 * nvec]
  __shared__ uint32_t s_ticket, s_moved;
  const int BG = g.B * g.Hkv;
  const int bg = (int)(blockIdx.x % (unsigned)BG);
  // per-(b, g) start-order ticket: a block only waits on items of its (b, g) that started before it
  if (threadIdx.x == 0) { s_ticket = atomicAdd(it.ticket + bg, 1u); s_moved = 0; }
  __syncthreads();
  const int item = (int)(s_ticket - it.ticket_base);
  const int4* rec = it.rec + (size_t)item * (1 + kMaintMoves);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = warp * kPerWarp + lane;
  // header and this lane's move record load together (records are padded to kMaintMoves)
  const int4 hd = rec[0];                                  // n_moves, dep_lo, dep_hi, phase
  const int4 mv = rec[1 + (lane < kPerWarp ? e : 0)];     // dst, ref, cand, inc
  const long long sbase = (long long)bg * g.S_tot;
  const double* mu = sd.mu + sbase;
  const float* s_bg = s + (long long)bg * (g.S_tot + g.m);
  const int nvec = g.d * (int)sizeof(T) / 16;             // vectors per K (or V) row

  int32_t my_dst = -1, my_src = 0;
  double my_mu = 0.0;
  int64_t my_org = 0;
  if (lane < kPerWarp && e < hd.x) {
    int32_t src = mv.y;
    if (src < 0) {
      if (it.inline_sel) {
        // winner of a depth-0 selection: cand if mu(cand) > mu(inc), strict (Q2); both
        // operands' mu and origin are loaded together
        const double mc = src_mu(g, mv.z, mu, s_bg), mi = src_mu(g, mv.w, mu, s_bg);
        const int64_t oc = mv.z < g.S_tot ? sd.origin[sbase + mv.z] : g.t0 + (mv.z - g.S_tot);
        const int64_t oi = mv.w < g.S_tot ? sd.origin[sbase + mv.w] : g.t0 + (mv.w - g.S_tot);
        const bool cw = mc > mi;
        src = cw ? mv.z : mv.w;
        my_mu = cw ? mc : mi;
        my_org = cw ? oc : oi;
      } else {
        src = p.resolved[(long long)bg * p.sel_cap + (-src - 1)];
        my_mu = src_mu(g, src, mu, s_bg);
        my_org = src < g.S_tot ? sd.origin[sbase + src] : g.t0 + (src - g.S_tot);
      }
    } else {
      my_mu = src_mu(g, src, mu, s_bg);                    // folded (Q9) or a new token's s
      my_org = src < g.S_tot ? sd.origin[sbase + src] : g.t0 + (src - g.S_tot);
    }
    if (src != mv.x) {                                     // resident won its selection: stays
      my_dst = mv.x;
      my_src = src;
    }
  }
  const uint32_t any = __ballot_sync(0xffffffffu, my_dst >= 0);
  const int gg = bg % g.Hkv, b = bg / g.Hkv;
#pragma unroll
  for (int j = 0; j < kPerWarp; ++j) {
    const int32_t sj = __shfl_sync(0xffffffffu, my_src, j);
    if (!((any >> j) & 1u)) continue;
    const T *ks, *vs;
    if (sj < g.S_tot) {
      ks = sd.k_raw + (sbase + sj) * g.d;
      vs = sd.v + (sbase + sj) * g.d;
    } else {                                               // a selection won by a chunk row
      const int r = sj - g.S_tot;
      ks = sd.k_in + (((long long)b * g.m + r) * g.Hkv + gg) * g.d;
      vs = sd.v_in + (((long long)b * g.m + r) * g.Hkv + gg) * g.d;
    }
    int4* row = s_rows + (warp * kPerWarp + j) * 2 * nvec;
    for (int i = lane; i < 2 * nvec; i += 32) {
      const int4* gsrc = i < nvec ? reinterpret_cast<const int4*>(ks) + i
                                  : reinterpret_cast<const int4*>(vs) + (i - nvec);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tc_smem_u32(row + i)), "l"(gsrc)
                   : "memory");
    }
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  // every loaded value must have ARRIVED before this block publishes, or a store of a later
  // item could overtake a load still in flight.  The rows are in shared memory (waited above);
  // the register operands are folded into one word that feeds the barrier's predicate
  // (consuming a register waits for its load).
  const uint32_t sink = (uint32_t)__double2loint(my_mu) ^ (uint32_t)my_org;
  __syncthreads_or(sink == 0x9E3779B9u);
  if (warp == 0) {
    if (lane == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(it.flags + (size_t)item * BG + bg), "r"(it.epoch)
                   : "memory");
    }
    // wait for the items that read this item's destinations (host-computed, all earlier)
    for (int j = hd.y + lane; j < hd.z; j += 32) {
      const uint32_t* f = it.flags + (size_t)j * BG + bg;
      uint32_t v;
      while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (v == it.epoch) break;
        __nanosleep(20);
      }
    }
  }
  __syncthreads();
  if (lane == 0 && any) atomicAdd(&s_moved, (uint32_t)__popc(any));
#pragma unroll
  for (int j = 0; j < kPerWarp; ++j) {
    const int32_t dj = __shfl_sync(0xffffffffu, my_dst, j);
    if (!((any >> j) & 1u)) continue;
    T* kd = sd.k_raw + (sbase + dj) * g.d;
    T* vd = sd.v + (sbase + dj) * g.d;
    const int4* row = s_rows + (warp * kPerWarp + j) * 2 * nvec;
    for (int i = lane; i < 2 * nvec; i += 32) {
      if (i < nvec) __stcs(reinterpret_cast<int4*>(kd) + i, row[i]);
      else __stcs(reinterpret_cast<int4*>(vd) + i - nvec, row[i]);
    }
  }
  if (my_dst >= 0) {
    sd.mu[sbase + my_dst] = my_mu;
    sd.origin[sbase + my_dst] = my_org;
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_moved) atomicAdd(it.moved + bg, (unsigned long long)s_moved);
}

// chunk_moves_kernel: moves that read no resident slot (chunk tokens entering C_1 or the sinks;
// selections between two chunk rows).  Launched after maint_kernel, so every resident read of
// the chunk is done; no ordering among them.  One warp per kChunkPerWarp (move, b*g) pairs, all
// loads in flight before the stores.
constexpr int kChunkPerWarp = 4;
template <typename T>
__global__ void __launch_bounds__(256) chunk_moves_kernel(Geometry g, PlanDev p, MaintItems it, StateDev<T> sd,
                                                          const float* __restrict__ s) {
  const int BG = g.B * g.Hkv;
  const int lane = threadIdx.x & 31;
  const int bg = blockIdx.y;
  const int w0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kChunkPerWarp;
  const float* s_bg = s + (long long)bg * (g.S_tot + g.m);
  const long long sbase = (long long)bg * g.S_tot;
  const int gg = bg % g.Hkv, b = bg / g.Hkv;
  const int nvec = g.d * (int)sizeof(T) / 16;
  int4 buf[kChunkPerWarp][2];
  int32_t dst[kChunkPerWarp], src[kChunkPerWarp];
#pragma unroll
  for (int u = 0; u < kChunkPerWarp; ++u) {
    const int e = w0 + u;
    dst[u] = -1;
    if (e >= it.n_chunk) continue;
    const int4 mv = it.chunk[e];                           // dst, ref, cand, inc
    int32_t sr = mv.y;
    if (sr < 0) {
      sr = it.inline_sel ? ((double)s_bg[mv.z] > (double)s_bg[mv.w] ? mv.z : mv.w)   // P:615, strict
                         : p.resolved[(long long)bg * p.sel_cap + (-sr - 1)];
    }
    dst[u] = mv.x; src[u] = sr;
    const int r = sr - g.S_tot;
    const int4* ks = reinterpret_cast<const int4*>(sd.k_in + (((long long)b * g.m + r) * g.Hkv + gg) * g.d);
    const int4* vs = reinterpret_cast<const int4*>(sd.v_in + (((long long)b * g.m + r) * g.Hkv + gg) * g.d);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = lane + 32 * h;
      if (i < nvec) buf[u][h] = __ldcs(ks + i);
      else if (i < 2 * nvec) buf[u][h] = __ldcs(vs + i - nvec);
    }
  }
#pragma unroll
  for (int u = 0; u < kChunkPerWarp; ++u) {
    if (dst[u] < 0) continue;
    int4* kd = reinterpret_cast<int4*>(sd.k_raw + (sbase + dst[u]) * g.d);
    int4* vd = reinterpret_cast<int4*>(sd.v + (sbase + dst[u]) * g.d);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = lane + 32 * h;
      if (i < nvec) __stcs(kd + i, buf[u][h]);
      else if (i < 2 * nvec) __stcs(vd + i - nvec, buf[u][h]);
    }
    if (lane == 0) {
      sd.mu[sbase + dst[u]] = (double)s_bg[src[u]];        // new token: mu = s
      sd.origin[sbase + dst[u]] = g.t0 + (src[u] - g.S_tot);
    }
  }
}

template <typename T>
void launch_maint(const Geometry& g, const PlanDev& p, const MaintItems& it, int n_items, StateDev<T> sd,
                  const float* s, cudaStream_t st) {
  const int BG = g.B * g.Hkv;
  if (n_items > 0) {
    const size_t smem = (size_t)kMaintMoves * 2 * g.d * sizeof(T);
    static bool attr_set[2] = {false, false};
    bool& done = attr_set[sizeof(T) == 2];
    if (!done) {   // full shared-memory carveout: 6 blocks of 32 KB per SM
      cudaFuncSetAttribute(maint_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      cudaFuncSetAttribute(maint_kernel<T>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      done = true;
    }
    maint_kernel<T><<<n_items * BG, 256, smem, st>>>(g, p, it, sd, s);
  }
  if (it.n_chunk > 0) {
    const int warps = (it.n_chunk + kChunkPerWarp - 1) / kChunkPerWarp;
    chunk_moves_kernel<T><<<dim3((warps + 7) / 8, BG), 256, 0, st>>>(g, p, it, sd, s);
  }
}

template void launch_maint<float>(const Geometry&, const PlanDev&, const MaintItems&, int, StateDev<float>,
                                  const float*, cudaStream_t);
template void launch_maint<__nv_bfloat16>(const Geometry&, const PlanDev&, const MaintItems&, int,
                                          StateDev<__nv_bfloat16>, const float*, cudaStream_t);

__global__ void positions_kernel(Geometry g, int32_t* __restrict__ pe) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < g.S_tot; x += gridDim.x * blockDim.x)
    pe[x] = slot_pe(g, x);
}

void launch_positions(const Geometry& g, int32_t* pe, cudaStream_t st) {
  int blocks = std::min(ceil_div(g.S_tot, 256), 148 * 4);
  positions_kernel<<<blocks, 256, 0, st>>>(g, pe);
}

}  // namespace cascade
