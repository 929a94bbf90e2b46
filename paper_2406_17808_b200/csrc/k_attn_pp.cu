// k_attn_pp.cu -- pass 1 (O and the row LSE of the strided-prefill slice, Fig. 4),
// two query tiles per CTA ("ping-pong"), d = 128.
//
// ncu on the 1-CTA kernel (k_attn_tc.cu) shows the MMA's shared-memory wavefronts at ~32 % of
// peak and the tensor pipe ~64 % active: the limiter is the chain softmax(j) -> PV(j) ->
// QK(j+2) of ONE softmax warp per SMSP (~580 instructions per 128-key tile).  Here a CTA owns
// query tiles A = 2x and B = 2x + 1 of one (b, q-head) against the SAME K/V tiles: while
// warpgroup A turns S_A into P_A, the tensor cores run B's QK^T / PV and vice versa, and each
// SMSP has two softmax warps.  K/V bytes per flop halve; Q moves to shared memory (A operand of
// an SS MMA) because TMEM holds S_A, S_B, O_A, O_B (4 x 128 columns); P_X overwrites the upper
// half of S_X, and QK_X(j+1) is issued after PV_X(j) (in-order tcgen05.mma).
//   warps 0-3  softmax of tile A, warps 4-7 softmax of tile B: the 1-CTA kernel's online
//              softmax (log2 domain, lazy 2^8 rescale, EMU of 16 exp2 pairs on the FMA pipe)
//   warp 8     TMA: both Q tiles once, then K/V tiles into a 2-stage ring
//   warp 9     TMEM allocator, then MMA: QK_A(0) QK_B(0) | PV_A(j) QK_A(j+1) PV_B(j) QK_B(j+1) ...
// (320 threads: 204 registers each, room for a 128-column S row without spilling)
#include <cuda.h>

#include "common.cuh"
#include "tc_util.cuh"

namespace cascade {

namespace {
constexpr int kPPTile = 128 * 128;   // one 128-row x 64-col bf16 block (16 KB)
}

template <int EMU>
__global__ void __launch_bounds__(320, 1)
attn_fwd_pp_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_vs, const __grid_constant__ CUtensorMap tm_vc, TcParams p,
                   int n_pairs) {
  constexpr int D = 128, KB = 2;
  constexpr int kStages = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;                                   // [2 tiles][KB blocks]
  uint8_t* sK = sQ + 2 * KB * kPPTile;                  // [kStages][KB blocks]
  uint8_t* sV = sK + kStages * KB * kPPTile;            // [kStages][KB blocks]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kStages * KB * kPPTile);
  uint64_t* kv_full = bars + 0;      // [2]
  uint64_t* kv_empty = bars + 2;     // [2]
  uint64_t* q_full = bars + 4;
  uint64_t* s_full = bars + 5;       // [A, B]
  uint64_t* p_full = bars + 7;       // [A, B]
  uint64_t* pv_done = bars + 9;      // [A, B]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 11);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // units: blocks [0, n_pairs) take query tiles (2x, 2x+1) of flat pair index u; the rest
  // split the remaining pairs into single tiles, so the pairs fill whole waves and the
  // half-cost singles the last one
  const int n_chunk_total = (p.m + 127) / 128;
  const int NP = (n_chunk_total + 1) / 2;               // tile pairs per (b, q-head)
  const int u = blockIdx.x;
  int fp, tA;
  bool hasB;
  if (u < n_pairs) {
    fp = u;
    tA = 2 * (fp % NP);
    hasB = tA + 1 < n_chunk_total;
  } else {
    const int sidx = u - n_pairs;
    fp = n_pairs + (sidx >> 1);
    tA = 2 * (fp % NP) + (sidx & 1);
    hasB = false;
  }
  const int h = (fp / NP) % p.Hq, b = (fp / NP) / p.Hq;
  const int gkv = h / p.G;
  const long long bg = (long long)b * p.Hkv + gkv;
  const int ntA = p.n_res_tiles + min(tA + 1, n_chunk_total);
  // B sees one more chunk tile than A; without B the K/V stream stops with A's tiles
  const int ntB = hasB ? p.n_res_tiles + min(tA + 2, n_chunk_total) : ntA;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) { tc::mbar_init(kv_full + i, 1); tc::mbar_init(kv_empty + i, 1); }
    tc::mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(s_full + i, 1); tc::mbar_init(p_full + i, 4); tc::mbar_init(pv_done + i, 1);
    }
    tc::fence_mbar_init();
  }
  if (warp == 8 && lane == 0) {
    tc::tma_prefetch(&tm_q); tc::tma_prefetch(&tm_k); tc::tma_prefetch(&tm_vs); tc::tma_prefetch(&tm_vc);
  }
  if (warp == 9) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ---------------- TMA producer ----------------
    if (tc::elect_one()) {
      const int qrow = (int)(((long long)b * p.Hq + h) * p.M + tA * 128);
      tc::mbar_expect_tx(q_full, (hasB ? 2 : 1) * KB * kPPTile);
      for (int x = 0; x < (hasB ? 2 : 1); ++x)
        for (int kb = 0; kb < KB; ++kb)
          tc::tma_load_2d(sQ + (x * KB + kb) * kPPTile, &tm_q, q_full, kb * 64, qrow + x * 128);
      for (int j = 0; j < ntB; ++j) {
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
        tc::mbar_expect_tx(kv_full + s, 2 * KB * kPPTile);
        for (int kb = 0; kb < KB; ++kb) {
          tc::tma_load_2d(sK + (s * KB + kb) * kPPTile, &tm_k, kv_full + s, kb * 64, krow);
          tc::tma_load_2d(sV + (s * KB + kb) * kPPTile, vm, kv_full + s, kb * 64, vrow);
        }
      }
    }
  } else if (warp == 9) {
    // ---------------- MMA issuer ----------------
    if (tc::elect_one()) {
      constexpr uint32_t idesc_qk = tc::idesc_bf16_f32(128, 128, 0);
      constexpr uint32_t idesc_pv = tc::idesc_bf16_f32(128, D, 1);
      const uint32_t aQ = tc::smem_u32(sQ), aK = tc::smem_u32(sK), aV = tc::smem_u32(sV);
      auto qk = [&](int x, int j) {                       // S_x = Q_x K_j^T
        const int s = j % kStages;
        tc::mbar_wait(kv_full + s, (j / kStages) & 1);
        tc::tc_fence_after();
        const uint32_t qbase = aQ + x * KB * kPPTile, kbase = aK + s * KB * kPPTile;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t da = tc::desc_kmajor_sw128(qbase + (kk >> 2) * kPPTile + (kk & 3) * 32);
          const uint64_t db = tc::desc_kmajor_sw128(kbase + (kk >> 2) * kPPTile + (kk & 3) * 32);
          tc::mma_bf16_ss(tmem + x * 128, da, db, idesc_qk, kk > 0 ? 1u : 0u);
        }
        tc::mma_commit(s_full + x);
      };
      auto pv = [&](int x, int j) {                       // O_x += P_x V_j
        tc::mbar_wait(p_full + x, j & 1);
        tc::tc_fence_after();
        const uint32_t vbase = aV + (j % kStages) * KB * kPPTile;
        const uint32_t pbase = tmem + x * 128 + 64;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {               // 128 keys = 8 x K16
          const uint64_t db = tc::desc_mnmajor_sw128(vbase + kk * 2048, kPPTile);
          tc::mma_bf16_ts(tmem + 256 + x * 128, pbase + kk * 8, db, idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit(pv_done + x);
      };
      tc::mbar_wait(q_full, 0);
      tc::tc_fence_after();
      qk(0, 0);
      if (hasB) qk(1, 0);
      for (int j = 0; j < ntB; ++j) {
        if (j < ntA) pv(0, j);
        if (j + 1 < ntA) qk(0, j + 1);
        if (hasB) pv(1, j);
        tc::mma_commit(kv_empty + (j % kStages));       // both PVs of tile j issued before it
        if (hasB && j + 1 < ntB) qk(1, j + 1);
      }
    }
  } else {
    // ---------------- softmax warpgroups: x = 0 (tile A), 1 (tile B) ----------------
    const int x = warp >> 2;
    const int nt = x == 0 ? ntA : (hasB ? ntB : 0);      // no B tile: its warps only wait at the end
    const int r = threadIdx.x & 127;                      // query row = TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int qi = (tA + x) * 128 + r;                    // chunk-relative query index
    const uint32_t sb = tmem + x * 128 + lane_off;
    const uint32_t ob = tmem + 256 + x * 128 + lane_off;
    float m_used = -INFINITY, l = 0.f;
    // S is read from TMEM in 64-column halves: columns 0-63 for the row max, then 64-127 (kept
    // in registers for the exp2 pass), then 0-63 again -- a thread holds 64 values, so 8
    // softmax warps fit the register file, with 3 TMEM-load waits per tile
    float xs[64];
    for (int j = 0; j < nt; ++j) {
      int lim;                                            // keys [0, lim) of the tile are visible
      if (j < p.n_res_tiles) {
        lim = p.res_tiles[j].y;
      } else {
        const int k0 = (j - p.n_res_tiles) * 128;
        lim = min(qi - k0 + 1, p.m - k0);
      }
      tc::mbar_wait(s_full + x, j & 1);
      tc::tc_fence_after();
      float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
      auto load_half = [&](int hf) {                      // columns [64 hf, 64 hf + 64) -> xs, masked
        tc::tmem_ld32(sb + hf * 64, xs);
        tc::tmem_ld32(sb + hf * 64 + 32, xs + 32);
        tc::tmem_wait_ld();
        if (lim < 128) {
#pragma unroll
          for (int e = 0; e < 64; ++e) xs[e] = hf * 64 + e < lim ? xs[e] : -INFINITY;
        }
      };
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        load_half(hf);
#pragma unroll
        for (int e = 0; e < 64; e += 4) {
          m0 = fmaxf(m0, xs[e]); m1 = fmaxf(m1, xs[e + 1]); m2 = fmaxf(m2, xs[e + 2]); m3 = fmaxf(m3, xs[e + 3]);
        }
      }
      const float mx = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)) * p.scale_log2;
      if (j == 0) {
        m_used = mx;
      } else {
        // lazy rescale of the O row when its max grew by more than 2^8 (see k_attn_tc.cu)
        const bool need = mx > m_used + 8.f;
        if (__any_sync(0xffffffffu, need)) {
          tc::mbar_wait(pv_done + x, (j - 1) & 1);
          tc::tc_fence_after();
          const float f = need ? tc::fast_exp2(m_used - mx) : 1.f;
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            float o[32];
            tc::tmem_ld32(ob + c * 32, o);
            tc::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] *= f;
            tc::tmem_st32(ob + c * 32, o);
          }
          if (need) { l *= f; m_used = mx; }
        }
      }
      const float mu = m_used == -INFINITY ? 0.f : m_used;
      const float2 sc2 = make_float2(p.scale_log2, p.scale_log2), nm2 = make_float2(-mu, -mu);
      float2 s0 = make_float2(0.f, 0.f), s1 = s0;
      // chunks 3, 2 from the registers (columns 64-127), then reload 0-63 for chunks 1, 0: P
      // chunk c lands on S columns [64 + 16 c, 80 + 16 c), which only chunks c' > c still read
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int c = 3 - cc;
        if (cc == 2) load_half(0);
        const float* xc = xs + (c & 1) * 32;
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float2 t = __ffma2_rn(make_float2(xc[2 * e], xc[2 * e + 1]), sc2, nm2);
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
      if (lane == 0) tc::mbar_arrive(p_full + x);
    }
    // epilogue
    if (nt > 0) {
    tc::mbar_wait(pv_done + x, (nt - 1) & 1);
    tc::tc_fence_after();
    const float inv = 1.f / l;
    const bool store = qi < p.m;
    __nv_bfloat16* orow = p.out + (((long long)b * p.m + qi) * p.Hq + h) * D;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      float o[32];
      tc::tmem_ld32(ob + c * 32, o);
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
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem);
  }
}

size_t attn_fwd_pp_smem() { return 1024 + (size_t)(2 * 2 + 2 * 2 * 2) * kPPTile + 12 * 8 + 64; }

void launch_attn_fwd_pp(const TcParams& p, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tvs,
                        const CUtensorMap& tvc, cudaStream_t st) {
  const int nq = (p.m + 127) / 128;
  const int total = p.B * p.Hq * ((nq + 1) / 2);        // tile pairs
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // the last partial wave of pairs runs as single tiles when they fit in one wave
  const int rem = total % sms;
  const int split = (total > sms && 2 * rem <= sms) ? rem : 0;
  const int n_pairs = total - split;
  const size_t smem = attn_fwd_pp_smem();
  auto kern = attn_fwd_pp_kernel<4>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<n_pairs + 2 * split, 320, smem, st>>>(tq, tk, tvs, tvc, p, n_pairs);
}

}  // namespace cascade
