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
//  2. maint_coop_kernel: ONE cooperative launch per chunk for all (b, g).  The host splits the
//     chunk's final moves {dst, ref, cand, inc} into "staged" moves that read a pre-chunk
//     resident slot (evictees carried to the next sub-cache, and selections,
//     P:611-619) and "chunk" moves that read only chunk rows.  The hazard is a staged move's
//     source being overwritten by another move of the same chunk, so staged rows are loaded
//     GPU-wide into shared memory (TMA bulk copies, selections resolved in place), all blocks
//     meet at one relaxed grid barrier, then the rows are bulk-stored; chunk moves (never
//     overwritten sources) fill the spare shared-memory rows and stream after the barrier.
//     A chunk whose staged moves exceed one round's shared memory runs several rounds, each
//     with its own barrier, in phase order (readers of a slot always precede its writer).
//
// All HBM-bound: 256-B rows moved by TMA bulk copies, mu / origin by the row's thread.
#include "common.cuh"
#include "tc_util.cuh"

#include <cstdio>
#include <cstdlib>
#include <vector>

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

// Homogeneous head policy: one decision per sequence.  Reduces each sequence's
// kv-head scores s[b, 0..Hkv) (already reduced over each GQA group) to one row -- max, or the
// mean of the group means (= the mean over all q-heads, the groups being equal) -- and writes it
// back to every kv-head, so every kv-head folds the same mu and takes the same selections.
__global__ void head_homogenize_kernel(int B, int Hkv, int len, int mode, float* __restrict__ s) {
  const long long total = (long long)B * len;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / len;
    const int x = (int)(i - b * len);
    float* sb = s + b * Hkv * (long long)len + x;
    float r = sb[0];
    for (int g = 1; g < Hkv; ++g) r = mode == 1 ? r + sb[(long long)g * len] : fmaxf(r, sb[(long long)g * len]);
    if (mode == 1) r = __fdiv_rn(r, (float)Hkv);
    for (int g = 0; g < Hkv; ++g) sb[(long long)g * len] = r;
  }
}

// Homogeneous policy with the median reduction (P:542 ablations): the median of every q-head's
// mass (numpy's convention for an even count: the mean of the middle two), written to every
// kv-head of the sequence.  Not a function of the per-kv-head reductions, so it reads the
// per-q-head masses the score producer wrote to `heads`.
__global__ void head_median_all_kernel(int B, int Hq, int Hkv, int len, const float* __restrict__ heads,
                                       int heads_ld, float* __restrict__ s) {
  const long long total = (long long)B * len;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / len;
    const int x = (int)(i - b * len);
    float hv[kMaxMedianGroup];
    for (int h = 0; h < Hq; ++h) hv[h] = heads[(b * Hq + h) * (long long)heads_ld + x];
    const float r = group_reduce_ablation(hv, Hq, 2);
    for (int g = 0; g < Hkv; ++g) s[(b * Hkv + g) * (long long)len + x] = r;
  }
}

void launch_head_median_all(int B, int Hq, int Hkv, int len, const float* heads, int heads_ld, float* s,
                            cudaStream_t st) {
  const long long total = (long long)B * len;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 8);
  head_median_all_kernel<<<blocks, 256, 0, st>>>(B, Hq, Hkv, len, heads, heads_ld, s);
}

void launch_head_homogenize(int B, int Hkv, int len, int mode, float* s, cudaStream_t st) {
  const long long total = (long long)B * len;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 8);
  head_homogenize_kernel<<<blocks, 256, 0, st>>>(B, Hkv, len, mode, s);
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

constexpr int kChunkPerWarp = 2;

// maint_coop_kernel: the whole chunk's moves in ONE cooperative launch, no per-item ordering.
// Moves that read a resident slot ("staged": evictees carried down a level, selections) are
// split into rounds of at most gridDim.x * rows-per-block (x) b*g pairs, in per-(b, g) phase
// order.  Round: every block loads its pairs' source rows into shared memory (cp.async) and
// their mu / origin (selections resolved here, strict '>'), grid barrier, stores them.
// Readers of a slot always come before its writer in phase order (they fill deeper
// sub-caches), so a slot written in round k was read in a round <= k, before that round's
// barrier.  Moves that read only chunk rows (never overwritten) fill the shared-memory rows the
// last round leaves free -- loaded with it, stored after its barrier -- and any excess streams
// through registers afterwards.
constexpr int kCoopThreads = 512;
// optional per-block timeline (globaltimer ns) for tuning: CASCADE_MAINT_TRACE=1
__device__ unsigned long long* g_maint_trace = nullptr;
__device__ __forceinline__ void trace_mark(int k) {
  if (g_maint_trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_maint_trace[blockIdx.x * 8 + k] = t;
  }
}
template <typename T, int VPL>
__global__ void __launch_bounds__(kCoopThreads, 2) maint_coop_kernel(Geometry g, PlanDev p, MaintItems it,
                                                                     StateDev<T> sd, const float* __restrict__ s) {
  extern __shared__ __align__(16) int4 s_rows[];          // [it.rows_per_block][2 * nvec]
  const int R = it.rows_per_block;
  double* s_mu = reinterpret_cast<double*>(s_rows + (size_t)R * 2 * (g.d * sizeof(T) / 16));
  int64_t* s_org = reinterpret_cast<int64_t*>(s_mu + R);
  long long* s_doff = reinterpret_cast<long long*>(s_org + R);   // destination flat row, -1: none
  __shared__ uint32_t s_moved;
  __shared__ __align__(8) uint64_t s_bar;                  // row loads of the current round
  const int BG = g.B * g.Hkv;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kWarps = kCoopThreads / 32;
  const uint32_t row_bytes = (uint32_t)(g.d * sizeof(T));  // one K (or V) row
  const int nvec = g.d * (int)sizeof(T) / 16;             // vectors per K (or V) row
  const uint32_t n = (uint32_t)it.n_staged, nc = (uint32_t)it.n_chunk;
  const uint32_t total = n * (uint32_t)BG;                // staged (move, b*g) pairs, b*g-major
  const uint32_t ctotal = nc * (uint32_t)BG;              // chunk-row pairs (both < 2^31)
  const uint32_t G = gridDim.x;
  const uint32_t per_round = G * (uint32_t)R;
  const uint32_t rounds = total ? (total + per_round - 1) / per_round : (ctotal ? 1u : 0u);
  if (threadIdx.x == 0) {
    s_moved = 0;
    tc::mbar_init(&s_bar, kCoopThreads);
    tc::fence_mbar_init();
  }
  __syncthreads();
  trace_mark(0);
  uint32_t bar = it.barrier_base;
  // grid barrier.  After a load phase only READS precede it, all complete (rows waited on, the
  // register operands stored to shared memory): a relaxed arrive suffices and no store can be
  // issued before the spin observes every arrival.  Between rounds it also orders the
  // previous round's stores (full fences).
  auto grid_barrier = [&](bool fenced) {
    __syncthreads();
    trace_mark(3);
    bar += G;
    if (threadIdx.x == 0) {
      if (fenced) __threadfence();
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(it.barrier) : "memory");
      uint32_t v;
      unsigned long long t_begin;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
      for (uint32_t spin = 0;; ++spin) {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(it.barrier) : "memory");
        if ((int32_t)(v - bar) >= 0) break;
        if ((spin & 1023u) == 1023u) {     // a barrier that cannot complete (a counter out of
          unsigned long long t;             // step with the host copy) traps after 10 s instead
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));   // of hanging the device
          if (t - t_begin > 10000000000ull) __trap();
        }
      }
      if (fenced) __threadfence();
    }
    __syncthreads();
  };
  // chunk-row pairs beyond the last round's spare rows ("overflow"): kChunkPerWarp per warp
  // through registers; the first batch is loaded before the last barrier and stored after it
  const uint32_t gw = blockIdx.x * kWarps + warp, nw = G * kWarps;
  int4 cbuf[kChunkPerWarp][VPL];
  int32_t cdst[kChunkPerWarp], csrc[kChunkPerWarp], cbg[kChunkPerWarp];
  auto chunk_load = [&](uint32_t w0) {
#pragma unroll
    for (int u = 0; u < kChunkPerWarp; ++u) {
      const uint32_t pi = w0 + u;
      cdst[u] = -1;
      if (pi >= ctotal) continue;
      const int bg = (int)(pi / nc);
      const int4 mv = it.chunk[pi - (uint32_t)bg * nc];
      const float* sbg = s + (long long)bg * (g.S_tot + g.m);
      int32_t sr = mv.y;
      if (sr < 0)
        sr = it.inline_sel ? ((double)sbg[mv.z] > (double)sbg[mv.w] ? mv.z : mv.w)   // P:615, strict
                           : p.resolved[(long long)bg * p.sel_cap + (-sr - 1)];
      cdst[u] = mv.x; csrc[u] = sr; cbg[u] = bg;
      const int r = sr - g.S_tot, gg = bg % g.Hkv, b = bg / g.Hkv;
      const int4* ks = reinterpret_cast<const int4*>(sd.k_in + (((long long)b * g.m + r) * g.Hkv + gg) * g.d);
      const int4* vs = reinterpret_cast<const int4*>(sd.v_in + (((long long)b * g.m + r) * g.Hkv + gg) * g.d);
#pragma unroll
      for (int h = 0; h < VPL; ++h) {
        const int i = lane + 32 * h;
        if (i < nvec) cbuf[u][h] = __ldcs(ks + i);
        else if (i < 2 * nvec) cbuf[u][h] = __ldcs(vs + i - nvec);
      }
    }
  };
  auto chunk_store = [&]() {
#pragma unroll
    for (int u = 0; u < kChunkPerWarp; ++u) {
      if (cdst[u] < 0) continue;
      const long long sb = (long long)cbg[u] * g.S_tot;
      int4* kd = reinterpret_cast<int4*>(sd.k_raw + (sb + cdst[u]) * g.d);
      int4* vd = reinterpret_cast<int4*>(sd.v + (sb + cdst[u]) * g.d);
#pragma unroll
      for (int h = 0; h < VPL; ++h) {
        const int i = lane + 32 * h;
        if (i < nvec) __stcs(kd + i, cbuf[u][h]);
        else if (i < 2 * nvec) __stcs(vd + i - nvec, cbuf[u][h]);
      }
      if (lane == 0) {
        sd.mu[sb + cdst[u]] = (double)s[(long long)cbg[u] * (g.S_tot + g.m) + csrc[u]];   // mu = s
        sd.origin[sb + cdst[u]] = g.t0 + (csrc[u] - g.S_tot);
      }
    }
  };
  // overflow pairs [ov0, ctotal): warp gw takes batches ov0 + (gw + k nw) kChunkPerWarp
  uint32_t ov0 = ctotal;
  // chunk-row pairs held in shared memory by the last round: cq per block
  uint32_t cq = 0;
  uint32_t moved = 0;
  for (uint32_t rd = 0; rd < rounds; ++rd) {
    const uint32_t r0 = rd * per_round;
    const bool last = rd + 1 == rounds;
    // this round's staged pairs, spread evenly over the blocks (<= R each)
    const uint32_t in_round = total > r0 ? min(per_round, total - r0) : 0u;
    const uint32_t q = (in_round + G - 1) / G;
    const uint32_t lo = r0 + blockIdx.x * q;
    const int cnt = (int)(blockIdx.x * q < in_round ? min(q, in_round - blockIdx.x * q) : 0u);
    int ccnt = 0;
    uint32_t clo = 0;
    if (last) {
      cq = min((uint32_t)R - q, (ctotal + G - 1) / G);
      clo = blockIdx.x * cq;
      ccnt = (int)(clo < ctotal ? min(cq, ctotal - clo) : 0u);
      ov0 = min(ctotal, G * cq);
      chunk_load(ov0 + gw * kChunkPerWarp);               // first overflow batch: loads in flight now
    }
    const int rows = cnt + ccnt;
    // phase A: one thread per row (rows <= blockDim) resolves its source (selections: strict
    // '>', Q2), loads mu / origin, and issues the row's two bulk copies (K, V) into
    // shared memory; every thread arrives once on the round's mbarrier
    {
      const int j = threadIdx.x;
      bool issued = false;
      if (j < rows) {
        const bool st = j < cnt;
        const uint32_t pi = st ? lo + (uint32_t)j : clo + (uint32_t)(j - cnt);
        const uint32_t nn = st ? n : nc;
        const int bg = (int)(pi / nn);
        const int4 mv = (st ? it.staged : it.chunk)[pi - (uint32_t)bg * nn];   // dst, ref, cand, inc
        const long long sb = (long long)bg * g.S_tot;
        const double* mu = sd.mu + sb;
        const float* sbg = s + (long long)bg * (g.S_tot + g.m);
        int32_t src = mv.y;
        if (src < 0) {
          if (it.inline_sel) {
            const bool cw = src_mu(g, mv.z, mu, sbg) > src_mu(g, mv.w, mu, sbg);
            src = cw ? mv.z : mv.w;
          } else {
            src = p.resolved[(long long)bg * p.sel_cap + (-src - 1)];
          }
        }
        const bool mv_row = src != mv.x;                   // resident won its selection: stays
        moved += (st && mv_row) ? 1u : 0u;                  // chunk-row moves: counted by the host
        s_doff[j] = mv_row ? sb + mv.x : -1;
        if (mv_row) {
          const T *ks, *vs;
          if (src < g.S_tot) {
            ks = sd.k_raw + (sb + src) * g.d;
            vs = sd.v + (sb + src) * g.d;
          } else {
            const int r = src - g.S_tot, gg = bg % g.Hkv, b = bg / g.Hkv;
            ks = sd.k_in + (((long long)b * g.m + r) * g.Hkv + gg) * g.d;
            vs = sd.v_in + (((long long)b * g.m + r) * g.Hkv + gg) * g.d;
          }
          uint8_t* row = reinterpret_cast<uint8_t*>(s_rows + (size_t)j * 2 * nvec);
          tc::mbar_expect_tx(&s_bar, 2 * row_bytes);
          tc::bulk_load(row, ks, row_bytes, &s_bar);
          tc::bulk_load(row + row_bytes, vs, row_bytes, &s_bar);
          issued = true;
          s_mu[j] = src_mu(g, src, mu, sbg);               // folded (Q9) or a new token's s
          s_org[j] = src < g.S_tot ? sd.origin[sb + src] : g.t0 + (src - g.S_tot);
        }
      }
      if (!issued) tc::mbar_arrive(&s_bar);
    }
    trace_mark(1);
    tc::mbar_wait(&s_bar, rd & 1u);
    trace_mark(2);
    if (total) grid_barrier(false);                        // every source of this round is read
    else __syncthreads();
    trace_mark(4);
    // phase B: the row's thread bulk-stores K and V from shared memory, then mu and origin
    tc::fence_proxy_async_smem();
    {
      const int j = threadIdx.x;
      if (j < rows && s_doff[j] >= 0) {
        const long long doff = s_doff[j];
        const uint8_t* row = reinterpret_cast<const uint8_t*>(s_rows + (size_t)j * 2 * nvec);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(sd.k_raw + doff * g.d),
                     "r"(tc::smem_u32(row)), "r"(row_bytes)
                     : "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(sd.v + doff * g.d),
                     "r"(tc::smem_u32(row + row_bytes)), "r"(row_bytes)
                     : "memory");
        sd.mu[doff] = s_mu[j];
        sd.origin[doff] = s_org[j];
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (last) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // smem stays valid
      else asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");            // writes done
    }
    if (last) chunk_store();
    else grid_barrier(true);                               // rows reused; stores ordered
  }
  // remaining overflow batches (the first one went with the last round)
  for (uint32_t w0 = ov0 + (gw + nw) * kChunkPerWarp; w0 < ctotal; w0 += nw * kChunkPerWarp) {
    chunk_load(w0);
    chunk_store();
  }
  if (moved) atomicAdd(&s_moved, moved);
  __syncthreads();
  trace_mark(5);
  if (threadIdx.x == 0 && s_moved) atomicAdd(it.moved + blockIdx.x % BG, (unsigned long long)s_moved);
}

template <typename T>
size_t maint_coop_smem(int d, int rows) {
  return (size_t)rows * 2 * d * sizeof(T) + (size_t)rows * (8 + 8 + 8) + 16;
}

// Grid of the cooperative maintenance launch: co-resident blocks (2 per SM) and the rows each
// stages per round.
template <typename T>
MaintGrid maint_coop_grid(int d) {
  static MaintGrid mg[2] = {};
  MaintGrid& m = mg[d == 128 ? 1 : 0];
  if (m.blocks) return m;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int rows = std::min(kCoopThreads, (int)((110 * 1024 - 16) / (2 * d * sizeof(T) + 24)));
  const size_t smem = maint_coop_smem<T>(d, rows);
  auto kern = maint_coop_kernel<T, 1>;
  if (2 * d * sizeof(T) / 16 > 32) kern = maint_coop_kernel<T, 2>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kCoopThreads, smem);
  m.blocks = std::max(1, std::min(per_sm, 2)) * sms;
  m.rows_per_block = rows;
  return m;
}

template <typename T>
cudaError_t launch_maint(const Geometry& g, const PlanDev& p, MaintItems it, StateDev<T> sd, const float* s,
                         cudaStream_t st) {
  if (it.n_staged <= 0 && it.n_chunk <= 0) return cudaSuccess;
  const MaintGrid mg = maint_coop_grid<T>(g.d);
  it.rows_per_block = mg.rows_per_block;
  const size_t smem = maint_coop_smem<T>(g.d, mg.rows_per_block);
  void* args[] = {(void*)&g, (void*)&p, (void*)&it, (void*)&sd, (void*)&s};
  const void* kern = 2 * g.d * sizeof(T) / 16 > 32 ? (const void*)maint_coop_kernel<T, 2>
                                                   : (const void*)maint_coop_kernel<T, 1>;
  static unsigned long long* trace = nullptr;
  static int trace_on = -1, trace_n = 0;
  if (trace_on < 0) {
    const char* e = std::getenv("CASCADE_MAINT_TRACE");
    trace_on = e && std::atoi(e) > 0 ? std::atoi(e) : 0;
    if (trace_on) {
      cudaMalloc(&trace, (size_t)mg.blocks * 8 * 8);
      cudaMemcpyToSymbol(g_maint_trace, &trace, sizeof(trace));
    }
  }
  const cudaError_t rc = cudaLaunchCooperativeKernel(kern, dim3(mg.blocks), dim3(kCoopThreads), args, smem, st);
  if (rc != cudaSuccess) return rc;
  if (trace_on && ++trace_n == trace_on) {     // dump the n-th launch: per-block marks, ns
    std::vector<unsigned long long> h((size_t)mg.blocks * 8);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < mg.blocks; ++b) t0 = std::min(t0, h[b * 8]);
    std::fprintf(stderr, "maint trace (staged %d chunk %d): block start A1 A2wait barrier_in barrier_out end\n",
                 it.n_staged, it.n_chunk);
    for (int b = 0; b < mg.blocks; b += 1)
      std::fprintf(stderr, "%d %llu %llu %llu %llu %llu %llu\n", b, h[b * 8] - t0, h[b * 8 + 1] - t0,
                   h[b * 8 + 2] - t0, h[b * 8 + 3] - t0, h[b * 8 + 4] - t0, h[b * 8 + 5] - t0);
  }
  return cudaSuccess;
}

template <typename T>
int maint_barriers(const Geometry& g, const MaintItems& it) {
  const MaintGrid mg = maint_coop_grid<T>(g.d);
  const long long total = (long long)it.n_staged * g.B * g.Hkv;
  const long long per_round = (long long)mg.blocks * mg.rows_per_block;
  const long long rounds = (total + per_round - 1) / per_round;
  return (int)(rounds > 0 ? 2 * rounds - 1 : 0) * mg.blocks;
}

template cudaError_t launch_maint<float>(const Geometry&, const PlanDev&, MaintItems, StateDev<float>, const float*,
                                  cudaStream_t);
template int maint_barriers<float>(const Geometry&, const MaintItems&);
template int maint_barriers<__nv_bfloat16>(const Geometry&, const MaintItems&);
template cudaError_t launch_maint<__nv_bfloat16>(const Geometry&, const PlanDev&, MaintItems, StateDev<__nv_bfloat16>,
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
