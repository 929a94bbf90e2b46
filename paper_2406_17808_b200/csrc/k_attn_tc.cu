// k_attn_tc.cu -- bf16 attention on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Pass 1 (attn_fwd_tc): O and the row LSE of the strided-prefill slice (Fig. 4):
//   chunk queries attend to every valid resident slot (key tiles from the host tile list)
//   and to the chunk's own keys causally.  One CTA = one (b, q-head, 128-query tile):
//     warp 0     TMA producer: Q once, then K/V tiles into a 2-stage ring
//     warp 1     MMA issuer (one elected thread): S = Q K^T into TMEM (two S buffers), then
//                O += P V into TMEM (P from shared memory)
//     warp 2     TMEM allocator
//     warps 4-7  softmax: thread r owns query row r (TMEM lane r); online softmax in the
//                log2 domain with lazy rescaling (O is rescaled in TMEM only when the row
//                max grows by more than 2^8), P written to shared memory as bf16 in the
//                SWIZZLE_128B K-major layout the MMA reads, epilogue O / l -> bf16, LSE.
// Pass 2 (attn_score_tc): the exact per-key mass of Alg. 3 (reading Q6) needs
//   the final LSE of every query row, so it is a second, key-stationary pass: one CTA =
//   one (b, kv-head, 128-key tile); S^T = K Q^T lands in TMEM with lane = key, so thread r
//   accumulates sum_r' w_r' exp2(S * scale*log2e - lse2_r') over query columns with no
//   atomics; the G q-heads of the group are reduced with max in registers.
//   w_r = (1 - gamma) gamma^(m-1-r) enters as log2(w_r) subtracted from lse2.
#include <cuda.h>

#include "common.cuh"
#include "tc_util.cuh"

#include <type_traits>
#include <vector>
#include <cstdio>

// exp2 pairs of every 16 evaluated on the FMA pipe (the rest on MUFU): pass 1 and pass 2
#ifndef CASCADE_FWD_EMU
#define CASCADE_FWD_EMU 4
#endif
#ifndef CASCADE_SCORE_EMU
#define CASCADE_SCORE_EMU 4
#endif

namespace cascade {

namespace {
constexpr int kTileBytes = 128 * 128;          // one 128-row x 64-col bf16 block (16 KB)
}

// Optional pass-1 wait accounting (build with CASCADE_NVCC_EXTRA=-DCASCADE_PASS1_TRACE): per
// CTA, clock64 cycles the MMA issuer spends waiting for K/V tiles and for P, and the softmax
// warp 4 spends waiting for S, plus the CTA's total; dumped by launch_attn_fwd_tc.
#ifdef CASCADE_PASS1_TRACE
__device__ unsigned long long* g_p1_trace = nullptr;
#define P1_T0() const long long _t0 = clock64()
#define P1_ACC(v) (v) += clock64() - _t0
#else
#define P1_T0()
#define P1_ACC(v)
#endif
// Optional pass-2 cycle accounting (CASCADE_NVCC_EXTRA=-DCASCADE_PASS2_TRACE): per CTA, math warp 4
// (lane 0) splits its item loop into barrier waits, TMEM-load waits and the rest; the MMA thread
// records its q_full and s_free waits; dumped by launch_attn_score_tc.
#ifdef CASCADE_PASS2_TRACE
__device__ unsigned long long* g_p2_trace = nullptr;
#define P2_T0() const long long _t2 = clock64()
#define P2_ACC(v) (v) += clock64() - _t2
#else
#define P2_T0()
#define P2_ACC(v)
#endif

// Pass 1.  Shared-memory bandwidth (128 B/clk/SM) is the binding resource of a 128x128 MMA
// with both operands in SMEM, so Q and P live in TMEM (A operand from TMEM, "TS" MMAs) and
// only K/V stream through SMEM (3-stage TMA ring).  TMEM columns: S0 [0,128), S1 [128,256),
// O [256, 256+D), Q [384, 384+D/2); P of tile j (bf16 pairs) overwrites the upper half of S_(j%2).
// MMA issue order QK(0) QK(1) PV(0) QK(2) PV(1) ...; tcgen05.mma from one thread execute in
// order, so QK(j+2) overwrites S_(j%2) only after PV(j) has read P(j) from it.
// EST (CASCADE_OPT_ONEPASS_SCORES): the paper's one-pass estimate of the per-key mass (Alg. 3,
// P:628-650) inside pass 1, so no pass 2 runs.  After tile j's softmax, row r's weight is
// a_r = C_EMA[r] / (l_r + l_r rho / gamma_) with gamma_ = j + 1 steps done and rho = nt - j - 1 left
// (l_r and P share the running max, so P / l_r is the max-independent ratio the paper
// normalises).  The column sum over the 128 rows, sum_r a_r P[r, key], is one more MMA: P (bf16,
// also written to shared memory in the SWIZZLE_128B row layout) read as the MN-major A operand
// [keys x rows] times B = [rows x 16] holding a_r split into bf16 hi + lo columns, into a 16-column
// TMEM accumulator (double-buffered); the softmax warps read tile j-1's column sums while tile j's
// MMAs run and atomically add them to s_heads.  K/V use a 2-stage ring to make room for the two
// P buffers (64 KB).
template <int D, int EMU, bool EST>
__global__ void __launch_bounds__(256, 1)
attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_vs, const __grid_constant__ CUtensorMap tm_vc,
                   TcParams p) {
  constexpr int KB = D / 64;                   // 64-element K blocks of a row
  constexpr int kStages = EST ? 2 : 3;
  constexpr uint32_t kColO = 256, kColQ = 384, kColCs = 448;   // EST: column sums at 448 / 464
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sK = smem;                                   // kStages x KB blocks
  uint8_t* sV = sK + kStages * KB * kTileBytes;         // kStages x KB blocks
  uint8_t* sPb = sV + kStages * KB * kTileBytes;        // EST: 2 x P [128 rows x 128 keys] SW128 (2 blocks)
  uint8_t* sB2 = sPb + (EST ? 2 * 2 * kTileBytes : 0);  // EST: 2 x [16 x 128] K-major SW128 (2 KB blocks)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB2 + (EST ? 2 * 4096 : 0));
  uint64_t* kv_full = bars + 0;      // [3]
  uint64_t* kv_empty = bars + 3;     // [3]
  uint64_t* s_full = bars + 6;       // [2]
  uint64_t* p_full = bars + 8;       // [2]
  uint64_t* q_full = bars + 10;
  uint64_t* pv_done[2] = {bars + 11, bars + 14};   // PV of tiles j with j % 2 == i
  uint64_t* cs_done = bars + 12;     // [2] EST: column sums of tile j in TMEM buffer j % 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 15);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int q0 = qt * 128;
  const int gkv = h / p.G;
  const long long bg = (long long)b * p.Hkv + gkv;
  const int n_chunk_tiles = min(q0 / 128 + 1, (p.m + 127) / 128);
  const int nt = p.n_res_tiles + n_chunk_tiles;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) { tc::mbar_init(kv_full + i, 1); tc::mbar_init(kv_empty + i, 1); }
    for (int i = 0; i < 2; ++i) { tc::mbar_init(s_full + i, 1); tc::mbar_init(p_full + i, 4); }
    tc::mbar_init(q_full, 4);
    tc::mbar_init(pv_done[0], 1);
    tc::mbar_init(pv_done[1], 1);
    tc::mbar_init(cs_done + 0, 1);
    tc::mbar_init(cs_done + 1, 1);
    tc::fence_mbar_init();
  }
  if (EST) {                                            // B operand rows 2..15 stay zero
    for (int o = threadIdx.x; o < 2 * 4096 / 16; o += blockDim.x) reinterpret_cast<uint4*>(sB2)[o] = make_uint4(0u, 0u, 0u, 0u);
    tc::fence_proxy_async_smem();
  }
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tm_k); tc::tma_prefetch(&tm_vs); tc::tma_prefetch(&tm_vc);
  }
  if (warp == 2) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer: K/V tiles ----------------
    if (tc::elect_one()) {
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
        tc::mbar_expect_tx(kv_full + s, 2 * KB * kTileBytes);
        uint8_t* k_dst = sK + s * KB * kTileBytes;
        uint8_t* v_dst = sV + s * KB * kTileBytes;
        for (int kb = 0; kb < KB; ++kb) {
          tc::tma_load_2d(k_dst + kb * kTileBytes, &tm_k, kv_full + s, kb * 64, krow);
          tc::tma_load_2d(v_dst + kb * kTileBytes, vm, kv_full + s, kb * 64, vrow);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (tc::elect_one()) {
      constexpr uint32_t idesc_qk = tc::idesc_bf16_f32(128, 128, 0);
      constexpr uint32_t idesc_pv = tc::idesc_bf16_f32(128, D, 1);
      const uint32_t aK = tc::smem_u32(sK), aV = tc::smem_u32(sV);
#ifdef CASCADE_PASS1_TRACE
      long long w_kv = 0, w_p = 0;
      const long long t_start = clock64();
#endif
      auto qk = [&](int j) {
        const int s = j % kStages;
        {
          P1_T0();
          tc::mbar_wait(kv_full + s, (j / kStages) & 1);
          P1_ACC(w_kv);
        }
        tc::tc_fence_after();
        const uint32_t kbase = aK + s * KB * kTileBytes;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t db = tc::desc_kmajor_sw128(kbase + (kk >> 2) * kTileBytes + (kk & 3) * 32);
          tc::mma_bf16_ts(tmem + (j & 1) * 128, tmem + kColQ + kk * 8, db, idesc_qk, kk > 0 ? 1u : 0u);
        }
        tc::mma_commit(s_full + (j & 1));
      };
      auto pv = [&](int j) {
        {
          P1_T0();
          tc::mbar_wait(p_full + (j & 1), (j >> 1) & 1);
          P1_ACC(w_p);
        }
        tc::tc_fence_after();
        const uint32_t vbase = aV + (j % kStages) * KB * kTileBytes;
        const uint32_t pbase = tmem + (j & 1) * 128 + 64;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {             // 128 keys = 8 x K16
          const uint64_t db = tc::desc_mnmajor_sw128(vbase + kk * 2048, kTileBytes);
          tc::mma_bf16_ts(tmem + kColO, pbase + kk * 8, db, idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
        }
        if (j + kStages < nt) tc::mma_commit(kv_empty + (j % kStages));   // the producer waits only these
        tc::mma_commit(pv_done[j & 1]);
        if (EST) {                                      // column sums sum_r a_r P[r, key]
          constexpr uint32_t idesc_cs = tc::idesc_bf16_f32(128, 16, 0, 1);   // A MN-major, B K-major
          const uint32_t pb = tc::smem_u32(sPb) + (j & 1) * 2 * kTileBytes;
          const uint32_t bb = tc::smem_u32(sB2) + (j & 1) * 4096;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {             // 128 rows = 8 x K16
            const uint64_t da = tc::desc_mnmajor_sw128(pb + kk * 2048, kTileBytes);
            const uint64_t db = tc::desc_kmajor_sw128(bb + (kk >> 2) * 2048 + (kk & 3) * 32);
            tc::mma_bf16_ss(tmem + kColCs + (j & 1) * 16, da, db, idesc_cs, kk > 0 ? 1u : 0u);
          }
          tc::mma_commit(cs_done + (j & 1));
        }
      };
      tc::mbar_wait(q_full, 0);
      tc::tc_fence_after();
      qk(0);
      if (nt > 1) qk(1);
      for (int j = 0; j < nt; ++j) {
        pv(j);
        if (j + 2 < nt) qk(j + 2);
      }
#ifdef CASCADE_PASS1_TRACE
      if (g_p1_trace) {
        const long long cta = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        g_p1_trace[cta * 6 + 0] = clock64() - t_start;
        g_p1_trace[cta * 6 + 1] = w_kv;
        g_p1_trace[cta * 6 + 2] = w_p;
        g_p1_trace[cta * 6 + 5] = nt;
      }
#endif
    }
  } else if (warp >= 4) {
    // ---------------- softmax warpgroup ----------------
    const int r = threadIdx.x - 128;                      // query row = TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int qi = q0 + r;                                // chunk-relative query index
    {   // Q row -> TMEM (A operand of every QK^T)
      const uint4* src = reinterpret_cast<const uint4*>(p.q_rot + (((long long)b * p.Hq + h) * p.M + qi) * D);
      const bool in_buf = qi < p.M;                       // rows past the scratch capacity: zeros
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {                 // 16 columns (32 bf16) per store
        uint32_t w[16];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const uint4 u = in_buf ? src[c * 4 + v] : make_uint4(0u, 0u, 0u, 0u);
          w[4 * v] = u.x; w[4 * v + 1] = u.y; w[4 * v + 2] = u.z; w[4 * v + 3] = u.w;
        }
        tc::tmem_st16(tmem + kColQ + lane_off + c * 16, w);
      }
      tc::tmem_wait_st();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(q_full);
    }
    float m_used = -INFINITY, l = 0.f;
    float x[128];
    // EST: tile jj's column sums (lane = key) -> s_heads[b][h][key] (atomic: every q-tile adds)
    auto est_readout = [&](int jj) {
      tc::mbar_wait_unbounded(cs_done + (jj & 1), (jj >> 1) & 1);
      tc::tc_fence_after();
      uint32_t cv[2];
      tc::tmem_ld_n<2>(tmem + kColCs + (jj & 1) * 16 + lane_off, cv);
      tc::tmem_wait_ld();
      const float v = __uint_as_float(cv[0]) + __uint_as_float(cv[1]);
      int key, len;
      if (jj < p.n_res_tiles) {
        const int2 t2 = p.res_tiles[jj];
        key = t2.x + r; len = t2.y;
      } else {
        const int k0 = (jj - p.n_res_tiles) * 128;
        key = p.S_tot + k0 + r; len = min(128, p.m - k0);
      }
      if (r < len && v != 0.f) atomicAdd(p.s_heads + ((long long)b * p.Hq + h) * (p.S_tot + p.Mb) + key, v);
    };
#ifdef CASCADE_PASS1_TRACE
    long long w_s = 0, w_pv = 0;
#endif
    for (int j = 0; j < nt; ++j) {
      const uint32_t sb = tmem + (j & 1) * 128 + lane_off;
      {
        P1_T0();
        tc::mbar_wait_unbounded(s_full + (j & 1), (j >> 1) & 1);
        P1_ACC(w_s);
      }
      tc::tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) tc::tmem_ld32(sb + c * 32, x + c * 32);
      tc::tmem_wait_ld();
      int lim;                                            // keys [0, lim) of the tile are visible
      if (j < p.n_res_tiles) {
        lim = p.res_tiles[j].y;
      } else {
        const int k0 = (j - p.n_res_tiles) * 128;
        lim = min(qi - k0 + 1, p.m - k0);
      }
      if (lim < 128) {                                    // mask only the (few) partial tiles
#pragma unroll
        for (int c = 0; c < 128; ++c) x[c] = c < lim ? x[c] : -INFINITY;
      }
      const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
      // exp2 of the tile against row offset mu -> P (bf16, TMEM) and its row sum; with TRACK,
      // the raw tile max is reduced alongside (ALU pipe, next to the MUFU / FMA work)
      auto exp_pass = [&](float mu, float& mraw, auto track) -> float {
        const float2 nm2 = make_float2(-mu, -mu);
        float2 s0 = make_float2(0.f, 0.f), s1 = s0;
        float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; ++c) {                     // 32 keys -> 16 packed columns per store
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float xa = x[c * 32 + 2 * e], xb = x[c * 32 + 2 * e + 1];
            if (decltype(track)::value) { m0 = fmaxf(m0, xa); m1 = fmaxf(m1, xb); }
            const float2 t = __ffma2_rn(make_float2(xa, xb), sc2, nm2);
            // EMU of every 16 pairs on the FMA pipe (degree-3 polynomial; P is rounded to bf16
            // anyway), the rest on MUFU
            const bool emu = ((e * EMU) % 16) + EMU >= 16;
            const float2 pp = emu ? tc::exp2_poly2<3>(t) : make_float2(tc::fast_exp2(t.x), tc::fast_exp2(t.y));
            if (e & 1) s1 = __fadd2_rn(s1, pp); else s0 = __fadd2_rn(s0, pp);
            pk[e] = tc::pack_bf16(pp.x, pp.y);
          }
          tc::tmem_st16(sb + 64 + c * 16, pk);
          if (EST) {                                      // the same bf16 P, row r, keys [32c, 32c + 32)
            uint8_t* prow = sPb + (j & 1) * 2 * kTileBytes + (c >> 1) * kTileBytes + r * 128;
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              const int ch = ((c & 1) * 4 + q4) ^ (r & 7);
              *reinterpret_cast<uint4*>(prow + ch * 16) =
                  make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
            }
          }
        }
        if (decltype(track)::value) mraw = fmaxf(m0, m1);
        const float2 s01 = __fadd2_rn(s0, s1);
        return s01.x + s01.y;
      };
      using Track = std::integral_constant<bool, true>;
      using NoTrack = std::integral_constant<bool, false>;
      float mraw = -INFINITY;
      if (j == 0) {
        // first tile: the row max first
        float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
#pragma unroll
        for (int c = 0; c < 128; c += 4) {
          m0 = fmaxf(m0, x[c]); m1 = fmaxf(m1, x[c + 1]); m2 = fmaxf(m2, x[c + 2]); m3 = fmaxf(m3, x[c + 3]);
        }
        m_used = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)) * p.scale_log2;
        l += exp_pass(m_used == -INFINITY ? 0.f : m_used, mraw, NoTrack{});
      } else {
        // later tiles: exp2 against the running max right away (P may reach 2^8 before a lazy
        // rescale, fine in fp32 / bf16); the tile max comes with it, and only if it grew by
        // more than 2^8 (rare) is O rescaled and the tile redone.  tcgen05.ld/st are
        // warp-collective, so the whole warp takes the branch if any row needs it; O must
        // hold every PV up to tile j-1 first.
        const float sum = exp_pass(m_used == -INFINITY ? 0.f : m_used, mraw, Track{});
        const float mx = mraw * p.scale_log2;
        const bool need = mx > m_used + 8.f;
        if (__any_sync(0xffffffffu, need)) {
          {
            P1_T0();
            tc::mbar_wait_unbounded(pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
            P1_ACC(w_pv);
          }
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
          tc::tmem_wait_st();                             // the first pass's P stores land first
          l += exp_pass(m_used == -INFINITY ? 0.f : m_used, mraw, NoTrack{});
        } else {
          l += sum;
        }
      }
      if (EST) {
        // a_r = C_EMA[r] / (l_r (1 + rho / gamma_)) = C_EMA[r] (j + 1) / (nt l_r), split into
        // bf16 hi + lo as columns 0 and 1 of the column-sum MMA's B operand (row r = K index r)
        const float a = (qi < p.m && l > 0.f) ? p.w[qi] * (float)(j + 1) / ((float)nt * l) : 0.f;
        const __nv_bfloat16 ah = __float2bfloat16_rn(a);
        const __nv_bfloat16 al = __float2bfloat16_rn(a - __bfloat162float(ah));
        uint8_t* b2 = sB2 + (j & 1) * 4096 + (r >> 6) * 2048;
        const int kc = (r & 63) >> 3, ke = (r & 7) * 2;
        *reinterpret_cast<__nv_bfloat16*>(b2 + 0 * 128 + ((kc ^ 0) << 4) + ke) = ah;
        *reinterpret_cast<__nv_bfloat16*>(b2 + 1 * 128 + ((kc ^ 1) << 4) + ke) = al;
        tc::fence_proxy_async_smem();
      }
      tc::tmem_wait_st();
      tc::tc_fence_before();
      // observe PV(j-1) (long done by now: it only needed P(j-1)), so every pv_done phase has a
      // waiter -- compute-sanitizer synccheck reports phases nobody waits for
      if (j >= 1) tc::mbar_wait_unbounded(pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(p_full + (j & 1));
      if (EST && j > 0) est_readout(j - 1);
    }
    if (EST && nt > 0) est_readout(nt - 1);
    // epilogue: O final once PV(nt-1) is done.  One barrier per PV parity: when this thread last
    // saw S(j) complete, QK(j) -- issued after PV(j-2) -- was done, so barrier j % 2 can only be
    // in the phase of PV(j) or past it and the parity wait is unambiguous.  (A single pv_done
    // could not tell PV(nt-1) done from PV(nt-3) done: with EST the cs_done wait above lets
    // PV(nt-1) finish first, and a parity wait for phase nt-2 then blocked forever.)  Both
    // barriers' phases are all waited (PV(j-1) at the end of tile j), none left unobserved.
    tc::mbar_wait_unbounded(pv_done[(nt - 1) & 1], ((nt - 1) >> 1) & 1);
#ifdef CASCADE_PASS1_TRACE
    if (g_p1_trace && threadIdx.x == 128) {
      const long long cta = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
      g_p1_trace[cta * 6 + 3] = w_s;
      g_p1_trace[cta * 6 + 4] = w_pv;
    }
#endif
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
    p.qbias[((long long)b * p.Hq + h) * p.Mb + qi] = store ? m_used + log2f(l) - p.log2w[qi] : INFINITY;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem);
  }
}

// 32 columns of one key row: acc += exp2(S * scale*log2e - b_q), packed f32x2 FMA/FADD,
// four independent accumulators.  CUT: column c only counts when c >= cut_from (query index
// >= key index inside the chunk's causal block).
template <bool CUT, int EMU, int DEG>
__device__ __forceinline__ void score_chunk(const float* x, const float* bq, float2 sc2, int cut_from,
                                            float2& a0, float2& a1, float2& a2, float2& a3) {
  const float4* b4 = reinterpret_cast<const float4*>(bq);
#pragma unroll
  for (int e = 0; e < 32; e += 4) {
    const float4 bb = b4[e >> 2];
    const float2 t0 = __ffma2_rn(make_float2(x[e], x[e + 1]), sc2, make_float2(-bb.x, -bb.y));
    const float2 t1 = __ffma2_rn(make_float2(x[e + 2], x[e + 3]), sc2, make_float2(-bb.z, -bb.w));
    // EMU of every 16 exp2 pairs on the FMA pipe (degree-DEG polynomial), the rest on MUFU
    const int q0i = (e >> 1), q1i = (e >> 1) + 1;           // pair indices 0..15 of this chunk
    const bool e0 = ((q0i * EMU) % 16) + EMU >= 16, e1 = ((q1i * EMU) % 16) + EMU >= 16;
    float2 p0 = e0 ? tc::exp2_poly2<DEG>(t0) : make_float2(tc::fast_exp2(t0.x), tc::fast_exp2(t0.y));
    float2 p1 = e1 ? tc::exp2_poly2<DEG>(t1) : make_float2(tc::fast_exp2(t1.x), tc::fast_exp2(t1.y));
    if (CUT) {
      p0.x = e + 0 >= cut_from ? p0.x : 0.f;
      p0.y = e + 1 >= cut_from ? p0.y : 0.f;
      p1.x = e + 2 >= cut_from ? p1.x : 0.f;
      p1.y = e + 3 >= cut_from ? p1.y : 0.f;
    }
    if ((e & 4) == 0) { a0 = __fadd2_rn(a0, p0); a1 = __fadd2_rn(a1, p1); }
    else { a2 = __fadd2_rn(a2, p0); a3 = __fadd2_rn(a3, p1); }
  }
}

// Pass 2: 20 warps, one CTA per PAIR of 128-key tiles (both tiles resident or both chunk
// tiles) so every Q tile fetched from L2 serves 256 keys.  warp 0 TMA (the two K tiles once,
// Q tiles through a 4-stage ring), warp 1 MMA (per item: S^T_w = K_w Q^T for w = 0, 1 into
// TMEM buffer 2*(i%2)+w), warp 2 TMEM allocator, warps 4-19 four math warpgroups: warpgroup
// (half, w) reads key tile w's S^T columns [64 half, 64 half + 64) (thread r = key r = TMEM
// lane r), so every SMSP has four exp2 warps to hide MUFU/TMEM latency.  Items are
// (q-head, q-tile); the two column halves meet in shared memory per head before the max.
template <int D, int EMU, int DEG>
__global__ void __launch_bounds__(640, 1)
attn_score_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     TcParams p) {
  constexpr int KB = D / 64;
  constexpr int kStages = 4;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sK = smem;                                   // 2 tiles x KB blocks (A operands)
  uint8_t* sQ = sK + 2 * KB * kTileBytes;               // kStages x KB blocks
  float* sb = reinterpret_cast<float*>(sQ + kStages * KB * kTileBytes);   // [kStages][128] q bias
  float* sacc = sb + kStages * 128;                     // [2 tiles][2 halves][G][128] partial sums
  uint64_t* bars = reinterpret_cast<uint64_t*>(sacc + 4 * p.G * 128);
  uint64_t* k_full = bars + 0;
  uint64_t* q_full = bars + 1;                 // [4]
  uint64_t* q_empty = bars + 5;                // [4]
  uint64_t* s_full = bars + 9;                 // [2]
  uint64_t* s_free = bars + 11;                // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 13);
  double* smu = reinterpret_cast<double*>(bars + 14);   // [2][128] EMA operands of the two key tiles

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid (b*g, pair): blocks launch x-fastest, so every (b, g)'s resident pairs go before the
  // cheaper causal chunk pairs and the last, partial wave is made of the cheap ones
  const int bgi = blockIdx.x;
  const int pair = blockIdx.y;
  const int b = bgi / p.Hkv, gkv = bgi - b * p.Hkv;
  const long long bg = bgi;
  // pair -> tiles: resident pairs first, then chunk pairs
  const int n_res_pairs = (p.n_res_tiles + 1) / 2;
  const int n_chunk_tiles = (p.m + 127) / 128;
  const bool resident = pair < n_res_pairs;
  int n_here, first;                                    // number of tiles in this pair, first tile
  if (resident) {
    first = 2 * pair;
    n_here = min(2, p.n_res_tiles - first);
  } else {
    first = 2 * (pair - n_res_pairs);                   // chunk tile index
    n_here = min(2, n_chunk_tiles - first);
  }
  const int nqt = n_chunk_tiles;
  const int qt_begin = resident ? 0 : first;            // q-tiles that can see the first chunk tile
  const int per_head = nqt - qt_begin;
  const int n_items = p.G * per_head;

  if (threadIdx.x == 0) {
    tc::mbar_init(k_full, 1);
    // a Q stage (tile + its 128 query biases) is free once the MMA read the tile (commit) and
    // the 8 math warps read the biases
    for (int i = 0; i < kStages; ++i) { tc::mbar_init(q_full + i, 1); tc::mbar_init(q_empty + i, 17); }
    for (int i = 0; i < 2; ++i) { tc::mbar_init(s_full + i, 1); tc::mbar_init(s_free + i, 16); }
    tc::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tc::tma_prefetch(&tm_q); tc::tma_prefetch(&tm_k); }
  if (warp == 2) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (tc::elect_one()) {
      tc::mbar_expect_tx(k_full, 2 * KB * kTileBytes);
      for (int w = 0; w < 2; ++w) {
        // a missing second tile loads the first again (never read back)
        const int t = first + min(w, n_here - 1);
        const int kstart = resident ? p.res_tiles[t].x : p.S_tot + t * 128;
        const int krow = (int)(bg * (p.S_tot + p.M) + kstart);
        for (int kb = 0; kb < KB; ++kb)
          tc::tma_load_2d(sK + (w * KB + kb) * kTileBytes, &tm_k, k_full, kb * 64, krow);
      }
      for (int i = 0, qi = 0, hi = 0; i < n_items; ++i) {
        const int st = i % kStages, u = i / kStages;
        if (i >= kStages) tc::mbar_wait(q_empty + st, (u - 1) & 1);
        const int hh = gkv * p.G + hi;
        const int q0 = (qt_begin + qi) * 128;
        if (++qi == per_head) { qi = 0; ++hi; }
        const int qrow = (int)(((long long)b * p.Hq + hh) * p.M + q0);
        tc::mbar_expect_tx(q_full + st, KB * kTileBytes + 512);
        for (int kb = 0; kb < KB; ++kb)
          tc::tma_load_2d(sQ + (st * KB + kb) * kTileBytes, &tm_q, q_full + st, kb * 64, qrow);
        tc::bulk_load(sb + st * 128, p.qbias + ((long long)b * p.Hq + hh) * p.Mb + q0, 512, q_full + st);
      }
    }
  } else if (warp == 1) {
    if (tc::elect_one()) {
      constexpr uint32_t idesc = tc::idesc_bf16_f32(128, 128, 0);
      const uint32_t aK = tc::smem_u32(sK), aQ = tc::smem_u32(sQ);
      tc::mbar_wait(k_full, 0);
#ifdef CASCADE_PASS2_TRACE
      long long w_q = 0, w_f = 0;
#endif
      for (int i = 0; i < n_items; ++i) {
        const int st = i % kStages, sb2 = i & 1;
        {
          P2_T0();
          tc::mbar_wait(q_full + st, (i / kStages) & 1);
          P2_ACC(w_q);
        }
        {
          P2_T0();
          if (i >= 2) tc::mbar_wait(s_free + sb2, ((i >> 1) - 1) & 1);
          P2_ACC(w_f);
        }
        tc::tc_fence_after();
        const uint32_t qb = aQ + st * KB * kTileBytes;
        for (int w = 0; w < n_here; ++w) {
          const uint32_t kbase = aK + w * KB * kTileBytes;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t da = tc::desc_kmajor_sw128(kbase + (kk >> 2) * kTileBytes + (kk & 3) * 32);
            const uint64_t db = tc::desc_kmajor_sw128(qb + (kk >> 2) * kTileBytes + (kk & 3) * 32);
            tc::mma_bf16_ss(tmem + (2 * sb2 + w) * 128, da, db, idesc, kk > 0 ? 1u : 0u);
          }
        }
        tc::mma_commit(s_full + sb2);
        tc::mma_commit(q_empty + st);
      }
#ifdef CASCADE_PASS2_TRACE
      if (g_p2_trace) {
        const long long cta = (long long)blockIdx.y * gridDim.x + blockIdx.x;
        g_p2_trace[cta * 8 + 3] = w_q;
        g_p2_trace[cta * 8 + 4] = w_f;
      }
#endif
    }
  } else if (warp == 3) {
    // EMA operands (mu) of the resident key tiles, staged for the epilogue's fold so the
    // math warps neither wait on HBM at the end nor hold them in registers
    if (resident && p.mu) {                              // mu null: the fold runs after (homogeneous)
      for (int w = 0; w < n_here; ++w) {
        const int2 tl = p.res_tiles[first + w];
        for (int j = lane; j < tl.y; j += 32) smu[w * 128 + j] = p.mu[bg * p.S_tot + tl.x + j];
      }
    }
    tc::named_bar_sync_roles(1, 544);
  } else if (warp >= 4) {
    const int wgi = (warp - 4) >> 2;                      // 0..3
    const int wg = wgi & 1, half = wgi >> 1;              // key tile of the pair, column half
    const int r = (threadIdx.x - 128) & 127;              // key row = TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const bool active = wg < n_here;
    const int t = first + wg;
    int kstart = 0, klen = 0, key_idx = 0;
    if (active) {
      if (resident) { kstart = p.res_tiles[t].x; klen = p.res_tiles[t].y; }
      else { kstart = p.S_tot + t * 128; klen = min(128, p.m - t * 128); key_idx = t * 128 + r; }
    }
    float* my_acc = sacc + (wg * 2 + half) * p.G * 128;
    for (int hh = 0; hh < p.G; ++hh) my_acc[hh * 128 + r] = 0.f;
    const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
    float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
    int qi = 0, hcur = 0;                                 // item i = (head hcur, q-tile qi), no division
#ifdef CASCADE_PASS2_TRACE
    long long w_bar = 0, w_ld = 0;
    const long long t_loop = clock64();
#endif
    for (int i = 0; i < n_items; ++i) {
      const int sb2 = i & 1, st = i % kStages;
      const int q0 = (qt_begin + qi) * 128 + half * 64;   // first query of this half
      const float* bq = sb + st * 128 + half * 64;
      {
        P2_T0();
        tc::mbar_wait(q_full + st, (i / kStages) & 1);    // biases of this item have landed
        tc::mbar_wait(s_full + sb2, (i >> 1) & 1);
        P2_ACC(w_bar);
      }
      tc::tc_fence_after();
      if (active) {
        const uint32_t tbase = tmem + (2 * sb2 + wg) * 128 + half * 64 + lane_off;
        const bool cut = !resident && q0 < (t + 1) * 128;   // causal cut inside this block
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float x[32];
          {
            P2_T0();
            tc::tmem_ld32(tbase + c * 32, x);
            tc::tmem_wait_ld();
            P2_ACC(w_ld);
          }
          if (!cut) score_chunk<false, EMU, DEG>(x, bq + c * 32, sc2, 0, a0, a1, a2, a3);
          else score_chunk<true, EMU, DEG>(x, bq + c * 32, sc2, key_idx - (q0 + c * 32), a0, a1, a2, a3);
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) { tc::mbar_arrive(s_free + sb2); tc::mbar_arrive(q_empty + st); }
      if (++qi == per_head) {                              // this half's sum for the head
        const float2 s01 = __fadd2_rn(a0, a1), s23 = __fadd2_rn(a2, a3);
        my_acc[hcur * 128 + r] = (s01.x + s01.y) + (s23.x + s23.y);
        a0 = a1 = a2 = a3 = make_float2(0.f, 0.f);
        qi = 0;
        ++hcur;
      }
    }
#ifdef CASCADE_PASS2_TRACE
    if (g_p2_trace && threadIdx.x == 128) {
      const long long cta = (long long)blockIdx.y * gridDim.x + blockIdx.x;
      g_p2_trace[cta * 8 + 0] = clock64() - t_loop;
      g_p2_trace[cta * 8 + 1] = w_bar;
      g_p2_trace[cta * 8 + 2] = w_ld;
      g_p2_trace[cta * 8 + 5] = n_items;
      g_p2_trace[cta * 8 + 6] = t_loop;
    }
#endif
    tc::named_bar_sync_roles(1, 544);                           // all halves' per-head sums in smem
    if (half == 0 && active && r < klen) {
      const float* h0 = sacc + (wg * 2 + 0) * p.G * 128;
      const float* h1 = sacc + (wg * 2 + 1) * p.G * 128;
      float best = 0.f;
      if (p.head_reduce == 0) {                           // max over the group
        for (int hh = 0; hh < p.G; ++hh) best = fmaxf(best, h0[hh * 128 + r] + h1[hh * 128 + r]);
      } else {                                            // mean / median ablations
        float hv[kMaxMedianGroup];
        for (int hh = 0; hh < p.G; ++hh) hv[hh] = h0[hh * 128 + r] + h1[hh * 128 + r];
        best = group_reduce_ablation(hv, p.G, p.head_reduce);
      }
      p.s[bg * (p.S_tot + p.m) + kstart + r] = best;
      if (p.heads_out)                                    // homogeneous + median: every head's mass
        for (int hh = 0; hh < p.G; ++hh)
          p.heads_out[((long long)b * p.Hq + gkv * p.G + hh) * (p.S_tot + p.Mb) + kstart + r] =
              h0[hh * 128 + r] + h1[hh * 128 + r];
      if (resident && p.mu)                               // EMA fold (Q4), never an FMA
        p.mu[bg * p.S_tot + kstart + r] = __dadd_rn(__dmul_rn(p.decay, smu[wg * 128 + r]), (double)best);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
#ifdef CASCADE_PASS2_TRACE
  if (g_p2_trace && threadIdx.x == 128) {
    const long long cta = (long long)blockIdx.y * gridDim.x + blockIdx.x;
    g_p2_trace[cta * 8 + 7] = clock64() - g_p2_trace[cta * 8 + 6];   // loop start -> CTA end
  }
#endif
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem);
  }
}

size_t attn_fwd_tc_smem(int d, bool est) {
  const int KB = d / 64;
  return est ? 1024 + (size_t)(2 * 2 * KB) * kTileBytes + 2 * 2 * kTileBytes + 2 * 4096 + 16 * 8 + 64
             : 1024 + (size_t)(2 * 3 * KB) * kTileBytes + 16 * 8 + 64;
}
size_t attn_score_tc_smem(int d, int G) {
  const int KB = d / 64;
  return 1024 + (size_t)(2 * KB + 4 * KB) * kTileBytes + 4 * 128 * 4 + (size_t)4 * G * 128 * 4 + 16 * 8 + 64 +
         2 * 128 * 8;
}

void launch_attn_fwd_tc(const TcParams& p, const CUtensorMap& tq, const CUtensorMap& tk,
                        const CUtensorMap& tvs, const CUtensorMap& tvc, int d, cudaStream_t st) {
  dim3 grid((p.m + 127) / 128, p.Hq, p.B);
  const bool est = p.s_heads != nullptr;
  const size_t smem = attn_fwd_tc_smem(d, est);
  // 4 of every 16 exp2 pairs on the FMA pipe: measured 75.1 / 78.3 / 78.4 / 76.0 % of peak for
  // 0 / 4 / 6 / 8 (scripts/kbench.py, steady state n_c = 62.5K)
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 256, smem, st>>>(tq, tk, tvs, tvc, p);
  };
#ifdef CASCADE_PASS1_TRACE
  static unsigned long long* trace = nullptr;
  static int calls = 0;
  const long long ctas = (long long)grid.x * grid.y * grid.z;
  if (!trace) {
    cudaMalloc(&trace, 8 * 6 * 4096LL * 64);
    cudaMemcpyToSymbol(g_p1_trace, &trace, sizeof(trace));
  }
#endif
  if (est) {
    if (d == 128) go(attn_fwd_tc_kernel<128, 4, true>);
    else go(attn_fwd_tc_kernel<64, 4, true>);
  } else {
    if (d == 128) go(attn_fwd_tc_kernel<128, CASCADE_FWD_EMU, false>);
    else go(attn_fwd_tc_kernel<64, 4, false>);
  }
#ifdef CASCADE_PASS1_TRACE
  if (++calls % 16 == 0 && ctas <= 4096LL * 64) {
    std::vector<unsigned long long> h(ctas * 6);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost);
    double a[6] = {0, 0, 0, 0, 0, 0};
    for (long long c = 0; c < ctas; ++c)
      for (int k = 0; k < 6; ++k) a[k] += (double)h[c * 6 + k];
    std::fprintf(stderr, "pass1 trace (call %d, %lld CTAs, %.1f tiles/CTA): per tile: CTA %.0f clk | MMA waits K/V %.0f, P %.0f | softmax waits S %.0f, PV(rescale) %.0f\n",
                 calls, ctas, a[5] / ctas, a[0] / a[5], a[1] / a[5], a[2] / a[5], a[3] / a[5], a[4] / a[5]);
  }
#endif
}

void launch_attn_score_tc(const TcParams& p, const CUtensorMap& tq, const CUtensorMap& tk, int d,
                          cudaStream_t st) {
  dim3 grid(p.B * p.Hkv, (p.n_res_tiles + 1) / 2 + ((p.m + 127) / 128 + 1) / 2);
  const size_t smem = attn_score_tc_smem(d, p.G);
  // exp2 pairs on the FMA pipe per 16: measured (degree-4 polynomial) 2.50 / 2.30 / 2.25 / 2.16 /
  // 2.20 / 2.21 / 2.44 ms per steady-state chunk for 0 / 2 / 3 / 4 / 5 / 6 / 8; after removing the
  // runtime divisions from the item loop, degree 4 at 4/16: 2.03 ms, degree 3 (7.5e-5 rel.) at
  // 3 / 4 / 5 of 16: 2.09 / 2.01 / 2.05 ms (scripts/kbench.py).  Prefetching both 32-column TMEM
  // chunks before the math (64 more live registers) measured 2.16 ms.
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 640, smem, st>>>(tq, tk, p);
  };
#ifdef CASCADE_PASS2_TRACE
  static unsigned long long* trace = nullptr;
  static int calls = 0;
  const long long ctas = (long long)grid.x * grid.y;
  if (!trace) {
    cudaMalloc(&trace, 8 * 8 * 16384LL);
    cudaMemcpyToSymbol(g_p2_trace, &trace, sizeof(trace));
  }
#endif
  if (d == 128) {
    go(attn_score_tc_kernel<128, CASCADE_SCORE_EMU, 3>);
  } else {
    go(attn_score_tc_kernel<64, CASCADE_SCORE_EMU, 3>);
  }
#ifdef CASCADE_PASS2_TRACE
  if (++calls % 16 == 0 && ctas <= 16384LL) {
    std::vector<unsigned long long> h(ctas * 8);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost);
    double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (long long c = 0; c < ctas; ++c)
      for (int k = 0; k < 8; ++k) if (k != 6) a[k] += (double)h[c * 8 + k];
    std::fprintf(stderr, "pass2 trace (call %d, %lld CTAs, %.1f items/CTA): per item: loop %.0f clk | math warp waits q/s_full %.0f, TMEM ld %.0f | MMA waits q_full %.0f, s_free %.0f | CTA loop->end %.0f clk/CTA\n",
                 calls, ctas, a[5] / ctas, a[0] / a[5], a[1] / a[5], a[2] / a[5], a[3] / a[5], a[4] / a[5], a[7] / ctas);
  }
#endif
}

// One-pass mode, after pass 1: s_g[key] = reduce_h s_heads[b][g G + h][key] over the group (max,
// P:542; mean / median ablations), and the EMA fold of the residents (mu <- decay mu + s_g, never
// an FMA) unless the homogeneous policy folds later.  One thread per (b, g, key) of the slot
// space [0, S_tot + m); empty slots keep s = 0.
__global__ void onepass_reduce_kernel(TcParams p, int32_t sink_pre, Geometry g, bool fold) {
  const long long total = (long long)p.B * p.Hkv * (p.S_tot + p.m);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long bg = i / (p.S_tot + p.m);
    const int x = (int)(i - bg * (p.S_tot + p.m));
    const int b = (int)(bg / p.Hkv), gg = (int)(bg - (long long)b * p.Hkv);
    bool valid = x >= p.S_tot || slot_pe(g, x) >= 0;
    if (!valid) continue;
    float hv[kMaxMedianGroup];
    float best = 0.f;
    for (int hh = 0; hh < p.G; ++hh) {
      const float v = p.s_heads[((long long)b * p.Hq + gg * p.G + hh) * (p.S_tot + p.Mb) + x];
      if (hh < kMaxMedianGroup) hv[hh] = v;
      best = fmaxf(best, v);
    }
    if (p.head_reduce) best = group_reduce_ablation(hv, p.G, p.head_reduce);
    p.s[bg * (p.S_tot + p.m) + x] = best;
    if (fold && x < p.S_tot)
      p.mu[bg * p.S_tot + x] = __dadd_rn(__dmul_rn(p.decay, p.mu[bg * p.S_tot + x]), (double)best);
  }
}

void launch_onepass_reduce(const TcParams& p, const Geometry& g, bool fold, cudaStream_t st) {
  const long long total = (long long)p.B * p.Hkv * (p.S_tot + p.m);
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 8);
  onepass_reduce_kernel<<<blocks, 256, 0, st>>>(p, g.sink_pre, g, fold);
}

}  // namespace cascade
