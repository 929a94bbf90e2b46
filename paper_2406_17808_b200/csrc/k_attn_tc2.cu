// k_attn_tc2.cu -- pass 1 (O and the row LSE of the strided-prefill slice, Fig. 4)
// on CTA pairs: tcgen05.mma.cta_group::2 with M = 256 (two 128-query tiles of one (b, q-head)).
//
// Why: with M = 128 a CTA stages 64 KB of K/V per 128-key tile through shared memory and its
// two MMAs read another 64 KB -- 128 KB per 1024 MMA cycles, the whole 128 B/clk shared-memory
// bandwidth of an SM.  In a CTA pair the B operands are split
// along N: CTA r loads keys [64 r, 64 r + 64) of each K tile (QK^T: N = keys) and head-dim
// columns [64 r, 64 r + 64) of each V tile (PV: N = d), so each SM stages and reads half.
//
// Roles per CTA (256 threads): warp 0 TMA producer (both CTAs; the peer's loads complete on
// the leader's barriers, `.cta_group::2`), warp 1 MMA issuer (leader CTA only), warp 2 TMEM
// allocator (both, cta_group::2), warps 4-7 softmax over the CTA's own 128 query rows -- the
// same online softmax with lazy rescale as the 1-CTA kernel (k_attn_tc.cu).  The peer's softmax
// arrives on the leader's q_full / p_full through shared::cluster addresses; the leader's
// commits multicast to both CTAs' s_full / pv_done / kv_empty.  Q is TMA-loaded into shared
// memory (A operand of an SS MMA; 32 KB more shared-memory reads per tile, still under the
// bandwidth); TMEM: S0 [0,128), S1 [128,256), O [384, 384+D); P of tile j over the upper half
// of S_(j%2).  The peer's arrivals are RELAXED cluster-scope mbarrier arrives issued after
// tcgen05.wait::st + tcgen05.fence::before_thread_sync: a release arrive costs a cluster-wide
// MEMBAR per tile on the critical path (measured 4.95 ms per steady-state chunk with release,
// 3.60 ms relaxed, vs 3.40 ms for the 1-CTA kernel).  A triple-buffered S broke parity and did
// not change the time.  Opt-in (CASCADE_FWD_PAIRS=1 at cascade_init) until it beats the 1-CTA
// kernel.
#include <cuda.h>

#include "common.cuh"
#include "tc_util.cuh"

namespace cascade {

namespace {

constexpr int kHalfBytes = 64 * 128;                  // 64 rows x 64 bf16 cols, SW128 (8 KB)
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;           // shared::cluster address -> CTA 0's copy

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the leader CTA's copy of a barrier (this CTA's shared address of the same object)
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(tc::smem_u32(bar)));
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ bool try_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(tc::smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t parity) {
  while (!try_wait_cluster(bar, parity)) {
  }
}
// 2D TMA load into this CTA's shared memory, bytes completing on the LEADER's barrier
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t x,
                                                 int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(tc::smem_u32(bar) & kPeerMask)
      : "memory");
}
__device__ __forceinline__ void mma2_bf16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma2_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on `bar` in both CTAs of the pair once this thread's MMAs have completed
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          tc::smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

}  // namespace

template <int EMU>
__global__ void __launch_bounds__(256, 1)
attn_fwd_tc2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k64,
                    const __grid_constant__ CUtensorMap tm_vs, const __grid_constant__ CUtensorMap tm_vc, TcParams p) {
  constexpr int D = 128;
  constexpr int kStages = 4;
  constexpr int kS = 2;                                   // S buffers in TMEM
  constexpr uint32_t kColO = 384;
  auto scol = [](int j) -> uint32_t { return (uint32_t)(j % kS) * 128u; };
  constexpr uint32_t kStageBytes = 2 * kHalfBytes + 128 * 128;   // K half (2 blocks) + V half (1 block)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + kStages * kStageBytes;             // this CTA's 128 x D query tile (2 blocks)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sQ + 2 * 128 * 128);
  uint64_t* kv_full = bars + 0;      // [kStages] leader: both CTAs' bytes
  uint64_t* kv_empty = bars + 4;     // [kStages] both (multicast commit)
  uint64_t* s_full = bars + 8;       // [3] both (multicast commit)
  uint64_t* p_full = bars + 11;      // [3] leader: 8 softmax warps of the pair
  uint64_t* q_full = bars + 14;      // leader: both CTAs' Q bytes
  uint64_t* pv_done = bars + 15;     // both (multicast commit)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int q0 = qt * 128;
  const int gkv = h / p.G;
  const long long bg = (long long)b * p.Hkv + gkv;
  // both CTAs run the pair's tile count (the odd tile sees one more chunk tile; the even one
  // masks it entirely)
  const int n_chunk_total = (p.m + 127) / 128;
  const int n_chunk_tiles = min((qt | 1) + 1, n_chunk_total);
  const int nt = p.n_res_tiles + n_chunk_tiles;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) { tc::mbar_init(kv_full + i, 1); tc::mbar_init(kv_empty + i, 1); }
    for (int i = 0; i < kS; ++i) { tc::mbar_init(s_full + i, 1); tc::mbar_init(p_full + i, 8); }
    tc::mbar_init(q_full, 1);
    tc::mbar_init(pv_done, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tm_q); tc::tma_prefetch(&tm_k64); tc::tma_prefetch(&tm_vs); tc::tma_prefetch(&tm_vc);
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tc::smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc::tc_fence_before();
  cluster_sync();                                         // barriers initialised in both CTAs
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs): this CTA's halves of K and V ----------------
    if (tc::elect_one()) {
      {   // this CTA's query tile (rows past the scratch capacity read as zeros: TMA bounds)
        const int qrow = (int)(((long long)b * p.Hq + h) * p.M + q0);
        if (leader) tc::mbar_expect_tx(q_full, 2 * 2 * 128 * 128);
        tma_load_2d_pair(sQ, &tm_q, q_full, 0, qrow);
        tma_load_2d_pair(sQ + 128 * 128, &tm_q, q_full, 64, qrow);
      }
      for (int j = 0; j < nt; ++j) {
        const int s = j % kStages, u = j / kStages;
        if (j >= kStages) tc::mbar_wait(kv_empty + s, (u - 1) & 1);
        int krow, vrow;
        const CUtensorMap* vm;
        if (j < p.n_res_tiles) {
          const int2 t = p.res_tiles[j];
          krow = (int)(bg * (p.S_tot + p.M) + t.x);
          vrow = (int)(bg * p.S_tot + t.x);
          vm = &tm_vs;
        } else {
          const int k0 = (j - p.n_res_tiles) * 128;
          krow = (int)(bg * (p.S_tot + p.M) + p.S_tot + k0);
          vrow = (int)(bg * p.M + k0);
          vm = &tm_vc;
        }
        if (leader) tc::mbar_expect_tx(kv_full + s, 2 * kStageBytes);   // both CTAs' bytes
        uint8_t* st = smem + s * kStageBytes;
        // K: keys [64 rank, 64 rank + 64) of the tile, both 64-column blocks of d
        tma_load_2d_pair(st, &tm_k64, kv_full + s, 0, krow + 64 * (int)rank);
        tma_load_2d_pair(st + kHalfBytes, &tm_k64, kv_full + s, 64, krow + 64 * (int)rank);
        // V: all 128 keys, head-dim columns [64 rank, 64 rank + 64)
        tma_load_2d_pair(st + 2 * kHalfBytes, vm, kv_full + s, 64 * (int)rank, vrow);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA) ----------------
    if (leader && tc::elect_one()) {
      constexpr uint32_t idesc_qk = tc::idesc_bf16_f32(256, 128, 0);
      constexpr uint32_t idesc_pv = tc::idesc_bf16_f32(256, D, 1);
      const uint32_t a0 = tc::smem_u32(smem), aQ = tc::smem_u32(sQ);
      auto qk = [&](int j) {
        const int s = j % kStages;
        wait_cluster(kv_full + s, (j / kStages) & 1);
        tc::tc_fence_after();
        const uint32_t kbase = a0 + s * kStageBytes;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t da = tc::desc_kmajor_sw128(aQ + (kk >> 2) * 128 * 128 + (kk & 3) * 32);
          const uint64_t db = tc::desc_kmajor_sw128(kbase + (kk >> 2) * kHalfBytes + (kk & 3) * 32);
          mma2_bf16_ss(tmem + scol(j), da, db, idesc_qk, kk > 0 ? 1u : 0u);
        }
        commit2(s_full + (j % kS));
      };
      auto pv = [&](int j) {
        wait_cluster(p_full + (j % kS), (j / kS) & 1);
        tc::tc_fence_after();
        const uint32_t vbase = a0 + (j % kStages) * kStageBytes + 2 * kHalfBytes;
        const uint32_t pbase = tmem + scol(j) + 64;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {             // 128 keys = 8 x K16
          const uint64_t db = tc::desc_mnmajor_sw128(vbase + kk * 2048, 128 * 128);
          mma2_bf16_ts(tmem + kColO, pbase + kk * 8, db, idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
        }
        commit2(kv_empty + (j % kStages));
        commit2(pv_done);
      };
      wait_cluster(q_full, 0);
      tc::tc_fence_after();
      for (int j = 0; j < kS && j < nt; ++j) qk(j);
      for (int j = 0; j < nt; ++j) {
        pv(j);
        if (j + kS < nt) qk(j + kS);
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax warpgroup (this CTA's 128 query rows) ----------------
    const int r = threadIdx.x - 128;                      // query row = TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int qi = q0 + r;                                // chunk-relative query index
    auto arrive = [&](uint64_t* bar) {
      if (leader) tc::mbar_arrive(bar);
      else arrive_leader(bar);
    };
    float m_used = -INFINITY, l = 0.f;
    float x[128];
    for (int j = 0; j < nt; ++j) {
      const uint32_t sb = tmem + scol(j) + lane_off;
      int lim;                                            // keys [0, lim) of the tile are visible
      if (j < p.n_res_tiles) {
        lim = p.res_tiles[j].y;
      } else {
        const int k0 = (j - p.n_res_tiles) * 128;
        lim = min(qi - k0 + 1, p.m - k0);
      }
      tc::mbar_wait(s_full + (j % kS), (j / kS) & 1);
      tc::tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) tc::tmem_ld32(sb + c * 32, x + c * 32);
      tc::tmem_wait_ld();
      float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
      if (lim < 128) {
#pragma unroll
        for (int c = 0; c < 128; ++c) x[c] = c < lim ? x[c] : -INFINITY;
      }
#pragma unroll
      for (int c = 0; c < 128; c += 4) {
        m0 = fmaxf(m0, x[c]); m1 = fmaxf(m1, x[c + 1]); m2 = fmaxf(m2, x[c + 2]); m3 = fmaxf(m3, x[c + 3]);
      }
      const float mx = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)) * p.scale_log2;
      if (j == 0) {
        m_used = mx;
      } else {
        // lazy rescale of the O row when its max grew by more than 2^8 (see k_attn_tc.cu)
        const bool need = mx > m_used + 8.f;
        if (__any_sync(0xffffffffu, need)) {
          tc::mbar_wait(pv_done, (j - 1) & 1);
          tc::tc_fence_after();
          const float f = need ? tc::fast_exp2(m_used - mx) : 1.f;
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            float o[32];
            tc::tmem_ld32(tmem + kColO + lane_off + c * 32, o);
            tc::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] *= f;
            tc::tmem_st32(tmem + kColO + lane_off + c * 32, o);
          }
          if (need) { l *= f; m_used = mx; }
        }
      }
      const float mu = m_used == -INFINITY ? 0.f : m_used;
      const float2 sc2 = make_float2(p.scale_log2, p.scale_log2), nm2 = make_float2(-mu, -mu);
      float2 s0 = make_float2(0.f, 0.f), s1 = s0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {                       // 32 keys -> 16 packed columns per store
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float2 t = __ffma2_rn(make_float2(x[c * 32 + 2 * e], x[c * 32 + 2 * e + 1]), sc2, nm2);
          const bool emu = ((e * EMU) % 16) + EMU >= 16;
          const float2 pp = emu ? tc::exp2_poly2<3>(t) : make_float2(tc::fast_exp2(t.x), tc::fast_exp2(t.y));
          if (e & 1) s1 = __fadd2_rn(s1, pp); else s0 = __fadd2_rn(s0, pp);
          pk[e] = tc::pack_bf16(pp.x, pp.y);
        }
        tc::tmem_st16(sb + 64 + c * 16, pk);
      }
      const float2 s01 = __fadd2_rn(s0, s1);
      l += s01.x + s01.y;
      tc::tmem_wait_st();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive(p_full + (j % kS));
    }
    // epilogue
    tc::mbar_wait(pv_done, (nt - 1) & 1);
    tc::tc_fence_after();
    const float inv = 1.f / l;
    const bool store = qi < p.m;
    __nv_bfloat16* orow = p.out + (((long long)b * p.m + qi) * p.Hq + h) * D;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      float o[32];
      tc::tmem_ld32(tmem + kColO + lane_off + c * 32, o);
      tc::tmem_wait_ld();
      if (store) {
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int v = 0; v < 4; ++v)
          dst[v] = make_uint4(tc::pack_bf16(o[8 * v + 0] * inv, o[8 * v + 1] * inv),
                              tc::pack_bf16(o[8 * v + 2] * inv, o[8 * v + 3] * inv),
                              tc::pack_bf16(o[8 * v + 4] * inv, o[8 * v + 5] * inv),
                              tc::pack_bf16(o[8 * v + 6] * inv, o[8 * v + 7] * inv));
      }
    }
    // pass-2 bias per query row: lse2 - log2(w_r); +inf for rows past m (they weigh nothing)
    if (qi < p.Mb)
      p.qbias[((long long)b * p.Hq + h) * p.Mb + qi] = store ? m_used + log2f(l) - p.log2w[qi] : INFINITY;
  }
  tc::tc_fence_before();
  cluster_sync();                                         // both CTAs done with the pair's TMEM
  if (warp == 2) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

size_t attn_fwd_tc2_smem() { return 1024 + (size_t)4 * (2 * kHalfBytes + 128 * 128) + 2 * 128 * 128 + 18 * 8 + 64; }

void launch_attn_fwd_tc2(const TcParams& p, const CUtensorMap& tq, const CUtensorMap& tk64, const CUtensorMap& tvs,
                         const CUtensorMap& tvc, cudaStream_t st) {
  const int nq = (p.m + 127) / 128;
  const size_t smem = attn_fwd_tc2_smem();
  auto kern = attn_fwd_tc2_kernel<4>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((nq + 1) / 2 * 2, p.Hq, p.B);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, tq, tk64, tvs, tvc, p);
}

}  // namespace cascade
