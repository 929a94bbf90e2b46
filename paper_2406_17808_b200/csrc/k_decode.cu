// k_decode.cu -- single-token step (Eq. 2) + its cascade update, bf16.
//
// Decode is HBM-bound (every cached K/V row is read once per step, ~4 flop/byte); the dot
// products still run on the tensor cores (tcgen05, M = 128 keys x N = 16 query columns) so the
// SIMT pipes are free for the per-key rotation and softmax:
//   decode_attn     grid (b*Hkv, split): TMA-fed, warp-specialised (below); each CTA streams a
//                   contiguous range of 128-slot key tiles, rotates every raw key in shared
//                   memory to its rank pe, S^T = K_rot Q^T and O^T += V^T P^T in TMEM,
//                   writes the log2-domain logits and the split's (max, sum, O).
//   decode_combine  one CTA per (b, q-head): merges the splits -> O (bf16) and lse2.
//   decode_update   one CTA per (b, g): exact mass s = w_0 * max_h exp2(logit_h - lse2_h)
//                   (Alg. 3 with m = 1: w_0 = 1 - gamma; max over the group), EMA fold
//                   mu <- gamma*mu + s for every resident, then Alg. 2's single
//                   insertion: the (at most one) selection and the (at most N+1) row moves,
//                   deepest sub-cache first.
#include "common.cuh"

#include <cmath>
#include "tc_util.cuh"

namespace cascade {

namespace {


}  // namespace

// Tensor-core decode attention (D = 128), TMA-fed and warp-specialised.  One CTA per
// (b*Hkv, split); the keys are the host's resident tile list (128-slot runs of one sub-cache,
// contiguous in memory) plus a 1-key tile for the new token.
//   warp 0     producer: TMA of the raw K tile (SWIZZLE_128B) + the cos/sin rows of the tile's
//              32-position blocks (bulk copies) into a 3-stage K ring, freed by QK^T
//   warp 3     producer: TMA of the V tile into a 3-stage V ring, freed by PV (split from the K
//              ring so K runs ahead of V: 0.924 -> 0.890 ms per configs[3] step)
//   warp 1     MMA: S^T[128 keys x 16] = K_rot Q^T (two S^T buffers, so QK(j+1) runs during
//              softmax(j)), then O^T[128 d x 16] += V^T P^T
//   warp 2     TMEM allocator
//   warps 4-7  softmax: thread t = key t: logits, online softmax per head, P^T
//   warps 8-15 two rotation warpgroups (half of the rotate-half pairs each): rotate every raw
//              key IN PLACE to its rank pe (cos/sin of (32a + b) theta by angle addition:
//              a-rows from the stage, b-rows resident), round to bf16 (reading Q17); they run
//              up to a full ring ahead of the softmax.
// Tile descriptor (int4, host): start slot, length, pe of key 0 (pe of key j = pe0 + j: the host
// splits a tile where a full ring wraps past its oldest slot).
namespace {
constexpr int kHiRows = 5;                                   // a-rows per tile: 128 consecutive pe span <= 5
constexpr int kLoRows = 32;                                  // pe = 32 a + b
constexpr int kLoStride = 64 * 8 + 8;                        // padded bytes per b-row (bank spread)
constexpr int kDecStages = 3;
}

template <int G>
__global__ void __launch_bounds__(512, 1) decode_attn_kernel(const __grid_constant__ CUtensorMap tm_k,
                                                             const __grid_constant__ CUtensorMap tm_v,
                                                             DecodeParams p) {
  constexpr int D = 128, HALF = 64;
  // K and V have separate rings: a K stage (32 KB + the tile's a-rows, padded to 1 KB for the next
  // stage's SWIZZLE_128B alignment) is free once QK^T has read it, a V stage (32 KB) once PV has
  constexpr int kKStageBytes = (32768 + kHiRows * 512 + 1023) / 1024 * 1024;
  constexpr int kVStageBytes = 32768;
  // All shared memory is dynamic (no static variables, so the window starts 1024-B aligned and
  // three stages fit): stages | Q | P | cos/sin(b theta) rows | small scalars and barriers.
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sK = dsm;                                        // kDecStages x [K | a-rows]
  uint8_t* sV = sK + kDecStages * kKStageBytes;             // kDecStages x V
  uint8_t* sQ = sV + kDecStages * kVStageBytes;             // [16 rows x 128 d] SW128 (2 x 2 KB)
  uint8_t* sP = sQ + 4096;                                  // [16 heads x 128 keys] SW128 (2 x 2 KB)
  uint8_t* sLo = sP + 4096;                                 // 32 x kLoStride: cos/sin(b theta_i)
  float (*sRed)[G] = reinterpret_cast<float (*)[G]>(sLo + kLoRows * kLoStride);   // [4][G]
  float* sCorr = reinterpret_cast<float*>(sRed + 4);
  int* sRescale = reinterpret_cast<int*>(sCorr + G);
  uint32_t* sTmemP = reinterpret_cast<uint32_t*>(sRescale + 1);
  uint64_t* bars = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(sTmemP + 1) + 7) & ~uintptr_t(7));
  uint64_t* kfull = bars + 0;       // [3]
  uint64_t* kempty = bars + 3;      // [3]
  uint64_t* rot_full = bars + 6;    // [3 stages][2 rotation warpgroups]
  uint64_t* s_full = bars + 12;     // [2] per S^T buffer
  uint64_t* p_full = bars + 14;     // [2] per S^T buffer
  uint64_t* pv_done = bars + 16;
  uint64_t* vfull = bars + 17;      // [3]
  uint64_t* vempty = bars + 20;     // [3]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bg = blockIdx.x, split = blockIdx.y;
  const int b = bg / p.Hkv, g = bg - b * p.Hkv;
  const int n_tiles = p.n_tiles + 1;                         // + the new-token tile
  const int per = (n_tiles + p.nsplit - 1) / p.nsplit;
  const int tbeg = split * per, tend = min(n_tiles, tbeg + per);
  const int nt = max(0, tend - tbeg);

  if (tid == 0) {
    for (int i = 0; i < kDecStages; ++i) {
      tc::mbar_init(kfull + i, 1); tc::mbar_init(kempty + i, 1);
      tc::mbar_init(vfull + i, 1); tc::mbar_init(vempty + i, 1);
    }
    for (int i = 0; i < 2 * kDecStages; ++i) tc::mbar_init(rot_full + i, 4);
    for (int i = 0; i < 2; ++i) { tc::mbar_init(s_full + i, 1); tc::mbar_init(p_full + i, 4); }
    tc::mbar_init(pv_done, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tc::tma_prefetch(&tm_k); tc::tma_prefetch(&tm_v); }
  if (warp == 2) tc::tmem_alloc<64>(sTmemP);
  // group queries rotated to pe = n_cached, bf16 (rows >= G zero); cos/sin(b theta) rows
  for (int o = tid; o < 16 * HALF; o += blockDim.x) {
    const int h = o / HALF, i = o - h * HALF;
    float r1 = 0.f, r2 = 0.f;
    if (h < G) {
      const __nv_bfloat16* qp = p.q + ((long long)b * p.Hq + g * G + h) * D;
      const double2 cs = p.tab[(long long)(p.n_keys - 1) * HALF + i];
      const double x1 = __bfloat162float(qp[i]), x2 = __bfloat162float(qp[i + HALF]);
      r1 = __double2float_rn(__dsub_rn(__dmul_rn(x1, cs.x), __dmul_rn(x2, cs.y)));
      r2 = __double2float_rn(__dadd_rn(__dmul_rn(x2, cs.x), __dmul_rn(x1, cs.y)));
    }
    const int off = h * 128 + ((((i >> 3) ^ (h & 7))) << 4) + (i & 7) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sQ + off) = __float2bfloat16_rn(r1);
    *reinterpret_cast<__nv_bfloat16*>(sQ + 2048 + off) = __float2bfloat16_rn(r2);
  }
  for (int o = tid; o < kLoRows * HALF; o += blockDim.x)
    *reinterpret_cast<float2*>(sLo + (o / HALF) * kLoStride + (o % HALF) * 8) = p.tab_lo[o];
  for (int o = tid; o < 4096 / 16; o += blockDim.x) reinterpret_cast<uint4*>(sP)[o] = make_uint4(0u, 0u, 0u, 0u);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *sTmemP, tO = tmem + 16;          // S^T buffers at columns 0 and 32

  // per-tile geometry (same on every warp): start slot, length, pe of key 0
  auto tile_info = [&](int ti, int& start, int& len, int& pe0) {
    if (ti < p.n_tiles) {
      const int4 t4 = p.dec_tiles[ti];
      start = t4.x; len = t4.y; pe0 = t4.z;
    } else {
      start = p.S_tot; len = 1; pe0 = p.n_keys - 1;              // the new token
    }
  };

  if (warp == 0) {
    if (tc::elect_one()) {
      for (int j = 0; j < nt; ++j) {              // K tiles + a-rows
        const int s = j % kDecStages;
        if (j >= kDecStages) tc::mbar_wait(kempty + s, ((j / kDecStages) - 1) & 1);
        int start, len, pe0;
        tile_info(tbeg + j, start, len, pe0);
        uint8_t* st = sK + s * kKStageBytes;
        // a-rows of the tile's pe range [pe0, pe0 + len)
        const int a0 = pe0 >> 5, nA = ((pe0 + len - 1) >> 5) - a0 + 1;
        const uint32_t bytes = (start < p.S_tot ? 32768u : 0u) + (uint32_t)nA * 512u;
        tc::mbar_expect_tx(kfull + s, bytes);
        if (start < p.S_tot) {
          const int row = (int)((long long)bg * p.S_tot + start);
          for (int kb = 0; kb < 2; ++kb) tc::tma_load_2d(st + kb * 16384, &tm_k, kfull + s, kb * 64, row);
        }
        for (int r = 0; r < nA; ++r) tc::bulk_load(st + 32768 + r * 512, p.tab_hi + (long long)(a0 + r) * HALF, 512, kfull + s);
      }
    }
  } else if (warp == 3) {
    if (tc::elect_one()) {
      for (int j = 0; j < nt; ++j) {              // V tiles (the new token's V is written by the rotation warps)
        const int s = j % kDecStages;
        if (j >= kDecStages) tc::mbar_wait(vempty + s, ((j / kDecStages) - 1) & 1);
        int start, len, pe0;
        tile_info(tbeg + j, start, len, pe0);
        uint8_t* st = sV + s * kVStageBytes;
        if (start < p.S_tot) {
          tc::mbar_expect_tx(vfull + s, 32768u);
          const int row = (int)((long long)bg * p.S_tot + start);
          for (int kb = 0; kb < 2; ++kb) tc::tma_load_2d(st + kb * 16384, &tm_v, vfull + s, kb * 64, row);
        } else {
          tc::mbar_arrive(vfull + s);             // stage free: the rotation warps may write it
        }
      }
    }
  } else if (warp == 1) {
    if (tc::elect_one()) {
      constexpr uint32_t idesc_qk = tc::idesc_bf16_f32(128, 16, 0, 0);
      constexpr uint32_t idesc_pv = tc::idesc_bf16_f32(128, 16, 0, 1);
      const uint32_t aQ = tc::smem_u32(sQ), aP = tc::smem_u32(sP);
      auto qk = [&](int j) {
        const int s = j % kDecStages;
        const uint32_t st = tc::smem_u32(sK + s * kKStageBytes);
        tc::mbar_wait(rot_full + 2 * s, (j / kDecStages) & 1);       // both rotated halves in place
        tc::mbar_wait(rot_full + 2 * s + 1, (j / kDecStages) & 1);
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t da = tc::desc_kmajor_sw128(st + (kk >> 2) * 16384 + (kk & 3) * 32);
          const uint64_t db = tc::desc_kmajor_sw128(aQ + (kk >> 2) * 2048 + (kk & 3) * 32);
          tc::mma_bf16_ss(tmem + (j & 1) * 32, da, db, idesc_qk, kk > 0 ? 1u : 0u);
        }
        tc::mma_commit(kempty + s);                  // K stage free once QK^T has read it
        tc::mma_commit(s_full + (j & 1));
      };
      if (nt > 0) qk(0);
      for (int j = 0; j < nt; ++j) {
        if (j + 1 < nt) qk(j + 1);                          // overlaps softmax(j)
        const int s = j % kDecStages;
        const uint32_t st = tc::smem_u32(sV + s * kVStageBytes);
        tc::mbar_wait(p_full + (j & 1), (j >> 1) & 1);       // P^T written (and O^T rescaled)
        tc::mbar_wait(vfull + s, (j / kDecStages) & 1);
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t da = tc::desc_mnmajor_sw128(st + kk * 2048, 16384);
          const uint64_t db = tc::desc_kmajor_sw128(aP + (kk >> 2) * 2048 + (kk & 3) * 32);
          tc::mma_bf16_ss(tO, da, db, idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit(pv_done);
        tc::mma_commit(vempty + s);
      }
    }
  } else if (warp >= 8) {
    // ---------------- rotation warpgroups ----------------
    const int t = (tid - 256) & 127;                         // key row of the tile
    const int rwg = (tid - 256) >> 7;                        // chunks [4 rwg, 4 rwg + 4)
    for (int j = 0; j < nt; ++j) {
      const int s = j % kDecStages;
      uint8_t* st = sK + s * kKStageBytes;
      int start, len, pe0;
      tile_info(tbeg + j, start, len, pe0);
      const bool valid = t < len;
      const int pe = pe0 + t;
      tc::mbar_wait(kfull + s, (j / kDecStages) & 1);
      if (start < p.S_tot) {
        // ---- rotate row t in place: pairs (i, i + 64) live at the same swizzled offset of the
        //      two 64-column blocks ----
        const int hr = (pe >> 5) - (pe0 >> 5);
        const float2* hi = reinterpret_cast<const float2*>(st + 32768 + (valid ? hr : 0) * 512);
        const float2* lo = reinterpret_cast<const float2*>(sLo + (pe & 31) * kLoStride);
#pragma unroll 2
        for (int c = 4 * rwg; c < 4 * rwg + 4; ++c) {
          const int off = t * 128 + ((c ^ (t & 7)) << 4);
          uint4* pa = reinterpret_cast<uint4*>(st + off);
          uint4* pb = reinterpret_cast<uint4*>(st + 16384 + off);
          const uint4 ua = *pa, ub = *pb;
          const uint32_t wa[4] = {ua.x, ua.y, ua.z, ua.w}, wb[4] = {ub.x, ub.y, ub.z, ub.w};
          uint32_t oa[4], ob[4];
#pragma unroll
          for (int e2 = 0; e2 < 4; ++e2) {
            float r[4];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int i = c * 8 + 2 * e2 + u;
              const float2 h2 = hi[i], l2 = lo[i];
              const float cs = h2.x * l2.x - h2.y * l2.y;  // cos((32a + b) theta_i)
              const float sn = h2.y * l2.x + h2.x * l2.y;  // sin((32a + b) theta_i)
              const float x1 = __uint_as_float(u ? (wa[e2] & 0xffff0000u) : (wa[e2] << 16));
              const float x2 = __uint_as_float(u ? (wb[e2] & 0xffff0000u) : (wb[e2] << 16));
              r[u] = x1 * cs - x2 * sn;
              r[2 + u] = x2 * cs + x1 * sn;
            }
            oa[e2] = tc::pack_bf16(r[0], r[1]);
            ob[e2] = tc::pack_bf16(r[2], r[3]);
          }
          *pa = make_uint4(oa[0], oa[1], oa[2], oa[3]);
          *pb = make_uint4(ob[0], ob[1], ob[2], ob[3]);
        }
      } else {
        // ---- the new token: key row 0 from the input, rotated to n_cached; rows >= 1 zero;
        //      its V row goes to the V stage once that is free ----
        tc::mbar_wait(vfull + s, (j / kDecStages) & 1);
        uint8_t* sv = sV + s * kVStageBytes;
        const int off_base = t * 128;
        for (int c = 4 * rwg; c < 4 * rwg + 4; ++c) {
          const int off = off_base + ((c ^ (t & 7)) << 4);
          uint4 ka = make_uint4(0u, 0u, 0u, 0u), kb2 = ka, va = ka, vb = ka;
          if (t == 0) {
            const uint4* kp = reinterpret_cast<const uint4*>(p.k_new + (long long)bg * D);
            const uint4* vp = reinterpret_cast<const uint4*>(p.v_new + (long long)bg * D);
            const uint4 ua = kp[c], ub = kp[8 + c];
            va = vp[c]; vb = vp[8 + c];
            const uint32_t wa[4] = {ua.x, ua.y, ua.z, ua.w}, wb[4] = {ub.x, ub.y, ub.z, ub.w};
            uint32_t oa[4], ob[4];
#pragma unroll
            for (int e2 = 0; e2 < 4; ++e2) {
              float r[4];
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                const int i = c * 8 + 2 * e2 + u;
                const double2 cs = p.tab[(long long)pe * HALF + i];
                const double x1 = __uint_as_float(u ? (wa[e2] & 0xffff0000u) : (wa[e2] << 16));
                const double x2 = __uint_as_float(u ? (wb[e2] & 0xffff0000u) : (wb[e2] << 16));
                r[u] = __double2float_rn(__dsub_rn(__dmul_rn(x1, cs.x), __dmul_rn(x2, cs.y)));
                r[2 + u] = __double2float_rn(__dadd_rn(__dmul_rn(x2, cs.x), __dmul_rn(x1, cs.y)));
              }
              oa[e2] = tc::pack_bf16(r[0], r[1]);
              ob[e2] = tc::pack_bf16(r[2], r[3]);
            }
            ka = make_uint4(oa[0], oa[1], oa[2], oa[3]);
            kb2 = make_uint4(ob[0], ob[1], ob[2], ob[3]);
          }
          *reinterpret_cast<uint4*>(st + off) = ka;
          *reinterpret_cast<uint4*>(st + 16384 + off) = kb2;
          *reinterpret_cast<uint4*>(sv + off) = va;
          *reinterpret_cast<uint4*>(sv + 16384 + off) = vb;
        }
      }
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(rot_full + 2 * s + rwg);
    }
  } else if (warp >= 4) {
    // ---------------- softmax warpgroup ----------------
    const int t = tid - 128;                                 // key = TMEM lane
    const int w4 = warp & 3;
    const uint32_t lane_off = (uint32_t)(w4 * 32) << 16;
    float m_run[G], l_part[G];
#pragma unroll
    for (int h = 0; h < G; ++h) { m_run[h] = -INFINITY; l_part[h] = 0.f; }
    for (int j = 0; j < nt; ++j) {
      int start, len, pe0;
      tile_info(tbeg + j, start, len, pe0);
      const bool valid = t < len;
      // ---- logits, block max per head, P^T ----
      tc::mbar_wait(s_full + (j & 1), (j >> 1) & 1);
      tc::tc_fence_after();
      float sv[16];
      tc::tmem_ld16(tmem + (j & 1) * 32 + lane_off, sv);
      tc::tmem_wait_ld();
      float lg[G];
#pragma unroll
      for (int h = 0; h < G; ++h) lg[h] = valid ? sv[h] * p.scale_log2 : -INFINITY;
      if (valid) {
        float* lp = p.logits + ((long long)bg * (p.S_tot + 1) + start + t) * G;
#pragma unroll
        for (int h = 0; h < G; ++h) lp[h] = lg[h];
      }
#pragma unroll
      for (int h = 0; h < G; ++h) {
        float v = lg[h];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) sRed[w4][h] = v;
      }
      tc::named_bar_sync(1, 128);
      if (t == 0) {
        int any = 0;
#pragma unroll
        for (int h = 0; h < G; ++h) {
          const float mt = fmaxf(fmaxf(sRed[0][h], sRed[1][h]), fmaxf(sRed[2][h], sRed[3][h]));
          const float mn = fmaxf(m_run[h], mt);
          const float cr = m_run[h] == -INFINITY ? 0.f : exp2f(m_run[h] - mn);
          sCorr[h] = cr;
          any |= (j > 0 && cr != 1.f);
          sRed[0][h] = mn;
        }
        *sRescale = any;
      }
      if (j >= 1) tc::mbar_wait(pv_done, (j - 1) & 1);      // sP free, O^T holds tiles < j
      tc::named_bar_sync(1, 128);
      tc::tc_fence_after();
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const float mn = sRed[0][h];
        const float cr = sCorr[h];
        m_run[h] = mn;
        const float pv = valid ? exp2f(lg[h] - mn) : 0.f;
        l_part[h] = l_part[h] * cr + pv;
        const int blk = t >> 6, kc = t & 63;
        *reinterpret_cast<__nv_bfloat16*>(sP + blk * 2048 + h * 128 + ((((kc >> 3) ^ (h & 7))) << 4) + (kc & 7) * 2) =
            __float2bfloat16_rn(pv);
      }
      if (*sRescale) {                                       // O^T column h *= corr_h (lane = d)
        float ov[16];
        tc::tmem_ld16(tO + lane_off, ov);
        tc::tmem_wait_ld();
#pragma unroll
        for (int h = 0; h < G; ++h) ov[h] *= sCorr[h];
        tc::tmem_st16(tO + lane_off, reinterpret_cast<const uint32_t*>(ov));
        tc::tmem_wait_st();
      }
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      tc::named_bar_sync(1, 128);                            // sRed / sCorr reads done
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(p_full + (j & 1));
    }
    // ---- split results ----
    {
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float v = l_part[h];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) sRed[w4][h] = v;
    }
    if (nt > 0) tc::mbar_wait(pv_done, (nt - 1) & 1);
    tc::tc_fence_after();
    tc::named_bar_sync(1, 128);
    const long long pbase = ((long long)bg * p.nsplit + split) * G;
    if (t < G) {
      p.part_ml[(pbase + t) * 2] = m_run[t];
      p.part_ml[(pbase + t) * 2 + 1] = sRed[0][t] + sRed[1][t] + sRed[2][t] + sRed[3][t];
    }
    float ov[16];
    tc::tmem_ld16(tO + lane_off, ov);
    tc::tmem_wait_ld();
#pragma unroll
    for (int h = 0; h < G; ++h) p.part_o[(pbase + h) * D + t] = nt > 0 ? ov[h] : 0.f;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc<64>(tmem);
  }
}

template <int D>
__global__ void decode_combine_kernel(DecodeParams p, __nv_bfloat16* __restrict__ out) {
  const int bh = blockIdx.x, d = threadIdx.x;
  const int b = bh / p.Hq, h = bh - b * p.Hq;
  const int g = h / p.G, j = h - g * p.G;
  const long long bg = (long long)b * p.Hkv + g;
  float M = -INFINITY;
  for (int s = 0; s < p.nsplit; ++s) M = fmaxf(M, p.part_ml[((bg * p.nsplit + s) * p.G + j) * 2]);
  float L = 0.f, o = 0.f;
  for (int s = 0; s < p.nsplit; ++s) {
    const long long base = (bg * p.nsplit + s) * p.G + j;
    const float ms = p.part_ml[base * 2];
    if (ms == -INFINITY) continue;
    const float f = exp2f(ms - M);
    L += p.part_ml[base * 2 + 1] * f;
    o += p.part_o[base * D + d] * f;
  }
  out[(long long)bh * D + d] = __float2bfloat16_rn(o / L);
  if (d == 0) p.lse2[bh] = M + log2f(L);
}

// One CTA per (b, g).  Plan (uploaded by the host): the m = 1 schedule of Alg. 2.
template <int D>
__global__ void __launch_bounds__(256) decode_update_kernel(DecodeParams p, PlanDev pl, int32_t n_sel,
                                                            const int32_t* __restrict__ phase_begin,
                                                            int32_t n_phase) {
  const int bg = blockIdx.x, tid = threadIdx.x;
  const int b = bg / p.Hkv, g = bg - b * p.Hkv;
  __shared__ float sl[16];
  if (tid < p.G) sl[tid] = p.lse2[(long long)b * p.Hq + g * p.G + tid];
  __syncthreads();
  double* mu = p.mu + (long long)bg * p.S_tot;
  float* s_out = p.s + (long long)bg * (p.S_tot + 1);
  const float* lg = p.logits + (long long)bg * (p.S_tot + 1) * p.G;
  // 1. exact mass + fold for every valid slot, run by run (sinks, C_1 .. C_N); the new token's
  //    mass lands at S_tot.  Empty slots keep s = 0 (zeroed when the layer was reset / init).
  const float4* lg4 = reinterpret_cast<const float4*>(lg);
  if (p.G == 4 && p.head_reduce == 0 && p.update_stage == 0) {
    // the common case (GQA 4:1, max): kU slots per thread in flight -- every logit / mu load of
    // the batch is issued before the first use, so the pass streams at HBM rate rather than at
    // one load round trip per slot
    constexpr int kU = 4;
    for (int run = 0; run <= p.N; ++run) {
      const int beg = run == 0 ? 0 : p.alpha + (run - 1) * p.c;
      const int len = run == 0 ? p.sink_pre : p.counts[run - 1];
      const int cap = run == 0 ? p.alpha : p.c;
      for (int o0 = tid; o0 < cap; o0 += kU * blockDim.x) {
        float4 l[kU];
        double m[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int o = o0 + u * blockDim.x;
          if (o < len) { l[u] = __ldcs(lg4 + beg + o); m[u] = mu[beg + o]; }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int o = o0 + u * blockDim.x, x = beg + o;
          if (o >= cap) continue;
          if (o >= len) { s_out[x] = 0.f; continue; }
          const float best = fmaxf(fmaxf(exp2f(l[u].x - sl[0]), exp2f(l[u].y - sl[1])),
                                   fmaxf(exp2f(l[u].z - sl[2]), exp2f(l[u].w - sl[3])));
          const float sv = p.w0 * best;
          s_out[x] = sv;
          mu[x] = __dadd_rn(__dmul_rn(p.decay, m[u]), (double)sv);
        }
      }
    }
  } else
  for (int run = 0; run <= p.N; ++run) {
    const int beg = run == 0 ? 0 : p.alpha + (run - 1) * p.c;
    const int len = run == 0 ? p.sink_pre : p.counts[run - 1];
    const int cap = run == 0 ? p.alpha : p.c;
    for (int o = tid; o < cap; o += blockDim.x) {
      const int x = beg + o;
      if (o >= len) { s_out[x] = 0.f; continue; }
      if (p.update_stage == 2) {                           // s already reduced (homogeneous)
        mu[x] = __dadd_rn(__dmul_rn(p.decay, mu[x]), (double)s_out[x]);
        continue;
      }
      float best = 0.f;
      if (p.head_reduce) {                                 // mean / median ablations
        float hv[kMaxMedianGroup];
        for (int h = 0; h < p.G; ++h) hv[h] = exp2f(lg[(long long)x * p.G + h] - sl[h]);
        best = group_reduce_ablation(hv, p.G, p.head_reduce);
      } else if (p.G == 4) {
        const float4 l = lg4[x];
        best = fmaxf(fmaxf(exp2f(l.x - sl[0]), exp2f(l.y - sl[1])), fmaxf(exp2f(l.z - sl[2]), exp2f(l.w - sl[3])));
      } else {
        for (int h = 0; h < p.G; ++h) best = fmaxf(best, exp2f(lg[(long long)x * p.G + h] - sl[h]));
      }
      const float sv = p.w0 * best;
      s_out[x] = sv;
      if (p.update_stage == 0) mu[x] = __dadd_rn(__dmul_rn(p.decay, mu[x]), (double)sv);
    }
  }
  if (tid == 0 && p.update_stage != 2) {
    float best = 0.f, hv[kMaxMedianGroup];
    for (int h = 0; h < p.G; ++h) {
      const float e = exp2f(lg[(long long)p.S_tot * p.G + h] - sl[h]);
      if (h < kMaxMedianGroup) hv[h] = e;           // G <= 32 whenever an ablation is on
      best = fmaxf(best, e);
    }
    if (p.head_reduce) best = group_reduce_ablation(hv, p.G, p.head_reduce);
    s_out[p.S_tot] = p.w0 * best;
  }
  if (p.update_stage == 1) return;                         // scores only (homogeneous, stage 1)
  __syncthreads();
  // 2. selections (depth order), 3. moves deepest sub-cache first -- one warp, sequential
  if (tid < 32) {
    int32_t* res = pl.resolved + (long long)bg * pl.sel_cap;
    if (tid == 0) {
      for (int jj = 0; jj < n_sel; ++jj) {
        const int k = pl.sel_order[jj];
        int32_t cand = pl.sel[3 * k + 1], inc = pl.sel[3 * k + 2];
        cand = cand >= 0 ? cand : res[-cand - 1];
        inc = inc >= 0 ? inc : res[-inc - 1];
        const double mc = cand < p.S_tot ? mu[cand] : (double)s_out[cand];
        const double mi = inc < p.S_tot ? mu[inc] : (double)s_out[inc];
        res[k] = mc > mi ? cand : inc;                    // strict '>'
      }
    }
    __syncwarp();
    for (int ph = 0; ph < n_phase; ++ph) {
      for (int e = phase_begin[ph]; e < phase_begin[ph + 1]; ++e) {
        const int32_t dst = pl.mov[2 * e];
        int32_t src = pl.mov[2 * e + 1];
        src = src >= 0 ? src : res[-src - 1];
        if (src == dst) continue;
        const __nv_bfloat16 *ks, *vs;
        double mu_new;
        int64_t org;
        if (src < p.S_tot) {
          ks = p.k_raw_mut + ((long long)bg * p.S_tot + src) * D;
          vs = p.v_mut + ((long long)bg * p.S_tot + src) * D;
          mu_new = mu[src];
          org = p.origin[(long long)bg * p.S_tot + src];
        } else {
          ks = p.k_new + (long long)bg * D;
          vs = p.v_new + (long long)bg * D;
          mu_new = (double)s_out[src];
          org = p.t0;
        }
        __nv_bfloat16* kd = p.k_raw_mut + ((long long)bg * p.S_tot + dst) * D;
        __nv_bfloat16* vd = p.v_mut + ((long long)bg * p.S_tot + dst) * D;
        constexpr int NV = D * 2 / 16;
        if (tid < NV) reinterpret_cast<uint4*>(kd)[tid] = reinterpret_cast<const uint4*>(ks)[tid];
        else if (tid < 2 * NV) reinterpret_cast<uint4*>(vd)[tid - NV] = reinterpret_cast<const uint4*>(vs)[tid - NV];
        if (tid == 0) { mu[dst] = mu_new; p.origin[(long long)bg * p.S_tot + dst] = org; }
        __syncwarp();
      }
    }
  }
}

size_t decode_attn_nsplit(const DecodeParams& p) {
  // splits per (b, g): minimise (waves of 1-CTA-per-SM CTAs) x (tiles per CTA + ~4 tiles of
  // per-CTA pipeline fill / combine overhead); >= 4 tiles per split.  Measured at B = 64,
  // Hkv = 8, 129 tiles (scripts/dbench.py): 1 / 2 / 3 / 4 / 5 / 6 / 8 / 12 splits ->
  // 1.010 / 0.922 / 0.968 / 0.954 / 0.985 / 0.984 / 1.014 / 1.066 ms per step; the model picks 2.
  const int bgs = p.B * p.Hkv;
  const int cap = std::max(1, std::min(64, (p.n_tiles + 1 + 3) / 4));
  int best = 1;
  double best_cost = 1e300;
  for (int ns = 1; ns <= cap; ++ns) {
    const double waves = std::ceil((double)bgs * ns / 148.0);
    const double cost = waves * ((double)(p.n_tiles + 1) / ns + 4.0);
    if (cost < best_cost) { best_cost = cost; best = ns; }
  }
  return (size_t)best;
}

template <int G>
void launch_attn(const DecodeParams& p, const CUtensorMap& tk, const CUtensorMap& tv, cudaStream_t st) {
  const size_t smem = kDecStages * ((32768 + kHiRows * 512 + 1023) / 1024 * 1024 + 32768) + 4096 + 4096 +
                      kLoRows * kLoStride + 4 * G * 4 + G * 4 + 8 + 8 + 23 * 8;
  cudaFuncSetAttribute(decode_attn_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  decode_attn_kernel<G><<<dim3(p.B * p.Hkv, p.nsplit), 512, smem, st>>>(tk, tv, p);
}

void launch_decode(const DecodeParams& p, const PlanDev& pl, int32_t n_sel, const int32_t* phase_begin_dev,
                   int32_t n_phase, __nv_bfloat16* out, const CUtensorMap& tk, const CUtensorMap& tv,
                   cudaStream_t st) {
  if (p.G == 4) launch_attn<4>(p, tk, tv, st);
  else if (p.G == 1) launch_attn<1>(p, tk, tv, st);
  else if (p.G == 2) launch_attn<2>(p, tk, tv, st);
  else launch_attn<8>(p, tk, tv, st);
  decode_combine_kernel<128><<<p.B * p.Hq, 128, 0, st>>>(p, out);
  if (!p.homogeneous) {
    decode_update_kernel<128><<<p.B * p.Hkv, 256, 0, st>>>(p, pl, n_sel, phase_begin_dev, n_phase);
    return;
  }
  // homogeneous head policy: every kv-head's s, then one reduction per sequence, then
  // the fold / selections / moves from the reduced s
  DecodeParams q = p;
  q.update_stage = 1;
  decode_update_kernel<128><<<p.B * p.Hkv, 256, 0, st>>>(q, pl, n_sel, phase_begin_dev, n_phase);
  launch_head_homogenize(p.B, p.Hkv, p.S_tot + 1, p.head_reduce, p.s, st);
  q.update_stage = 2;
  decode_update_kernel<128><<<p.B * p.Hkv, 256, 0, st>>>(q, pl, n_sel, phase_begin_dev, n_phase);
}

}  // namespace cascade
