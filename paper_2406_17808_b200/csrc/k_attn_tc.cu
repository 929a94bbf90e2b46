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

namespace cascade {

namespace {
constexpr int kTileBytes = 128 * 128;          // one 128-row x 64-col bf16 block (16 KB)
}

template <int D>
__global__ void __launch_bounds__(256, 1)
attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_vs, const __grid_constant__ CUtensorMap tm_vc,
                   TcParams p) {
  constexpr int KB = D / 64;                   // 64-element K blocks of a row
  constexpr int kStages = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                                   // KB blocks
  uint8_t* sP = sQ + KB * kTileBytes;                   // 2 blocks (128 keys)
  uint8_t* sK = sP + 2 * kTileBytes;                    // kStages x KB blocks
  uint8_t* sV = sK + kStages * KB * kTileBytes;         // kStages x KB blocks
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kStages * KB * kTileBytes);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;      // [2]
  uint64_t* kv_empty = bars + 3;     // [2]
  uint64_t* s_full = bars + 5;       // [2]
  uint64_t* s_free = bars + 7;       // [2]
  uint64_t* p_full = bars + 9;
  uint64_t* pv_done = bars + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int q0 = qt * 128;
  const int gkv = h / p.G;
  const long long bg = (long long)b * p.Hkv + gkv;
  const int n_chunk_tiles = min(q0 / 128 + 1, (p.m + 127) / 128);
  const int nt = p.n_res_tiles + n_chunk_tiles;

  if (threadIdx.x == 0) {
    tc::mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(kv_full + i, 1); tc::mbar_init(kv_empty + i, 1);
      tc::mbar_init(s_full + i, 1); tc::mbar_init(s_free + i, 4);
    }
    tc::mbar_init(p_full, 4);
    tc::mbar_init(pv_done, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tm_q); tc::tma_prefetch(&tm_k); tc::tma_prefetch(&tm_vs); tc::tma_prefetch(&tm_vc);
  }
  if (warp == 2) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS[2] = {tmem + 0, tmem + 128};
  const uint32_t tO = tmem + 256;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (tc::elect_one()) {
      const int qrow = (int)(((long long)b * p.Hq + h) * p.M + q0);
      tc::mbar_expect_tx(q_full, KB * kTileBytes);
      for (int kb = 0; kb < KB; ++kb) tc::tma_load_2d(sQ + kb * kTileBytes, &tm_q, q_full, kb * 64, qrow);
      for (int j = 0; j < nt; ++j) {
        const int s = j & 1, u = j >> 1;
        if (j >= 2) tc::mbar_wait(kv_empty + s, (u - 1) & 1);
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
      const uint32_t aQ = tc::smem_u32(sQ), aP = tc::smem_u32(sP);
      const uint32_t aK = tc::smem_u32(sK), aV = tc::smem_u32(sV);
      auto issue_pv = [&](int i) {
        tc::mbar_wait(p_full, i & 1);
        tc::tc_fence_after();
        const uint32_t vbase = aV + (i & 1) * KB * kTileBytes;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {             // 128 keys = 8 x K16
          const uint64_t da = tc::desc_kmajor_sw128(aP + (kk >> 2) * kTileBytes + (kk & 3) * 32);
          const uint64_t db = tc::desc_mnmajor_sw128(vbase + kk * 2048, kTileBytes);
          tc::mma_bf16_ss(tO, da, db, idesc_pv, (i > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit(pv_done);
        tc::mma_commit(kv_empty + (i & 1));
      };
      tc::mbar_wait(q_full, 0);
      for (int j = 0; j < nt; ++j) {
        const int s = j & 1, u = j >> 1;
        tc::mbar_wait(kv_full + s, u & 1);
        if (j >= 2) tc::mbar_wait(s_free + s, (u - 1) & 1);
        tc::tc_fence_after();
        const uint32_t kbase = aK + s * KB * kTileBytes;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t da = tc::desc_kmajor_sw128(aQ + (kk >> 2) * kTileBytes + (kk & 3) * 32);
          const uint64_t db = tc::desc_kmajor_sw128(kbase + (kk >> 2) * kTileBytes + (kk & 3) * 32);
          tc::mma_bf16_ss(tS[s], da, db, idesc_qk, kk > 0 ? 1u : 0u);
        }
        tc::mma_commit(s_full + s);
        if (j >= 1) issue_pv(j - 1);
      }
      issue_pv(nt - 1);
    }
  } else if (warp >= 4) {
    // ---------------- softmax warpgroup ----------------
    const int r = threadIdx.x - 128;                      // query row = TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int qi = q0 + r;                                // chunk-relative query index
    float m_used = -INFINITY, l = 0.f;
    float x[128];
    for (int j = 0; j < nt; ++j) {
      const int s = j & 1, u = j >> 1;
      tc::mbar_wait(s_full + s, u & 1);
      tc::tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) tc::tmem_ld32(tS[s] + lane_off + c * 32, x + c * 32);
      tc::tmem_wait_ld();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(s_free + s);
      // mask + scale (log2 domain)
      int lim;                                            // keys [0, lim) of the tile are visible
      if (j < p.n_res_tiles) {
        lim = p.res_tiles[j].y;
      } else {
        const int k0 = (j - p.n_res_tiles) * 128;
        lim = min(qi - k0 + 1, p.m - k0);
      }
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 128; ++c) {
        x[c] = c < lim ? x[c] * p.scale_log2 : -INFINITY;
        mx = fmaxf(mx, x[c]);
      }
      if (j >= 1) {
        tc::mbar_wait(pv_done, (j - 1) & 1);              // O current, P buffer free
        tc::tc_fence_after();
        // Lazy rescale of the O row when its max grew by more than 2^8.  tcgen05.ld/st are
        // warp-collective (.sync.aligned), so the whole warp takes the branch if any row needs it.
        const bool need = mx > m_used + 8.f;
        if (__any_sync(0xffffffffu, need)) {
          const float f = need ? tc::fast_exp2(m_used - mx) : 1.f;
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            float o[32];
            tc::tmem_ld32(tO + lane_off + c * 32, o);
            tc::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] *= f;
            tc::tmem_st32(tO + lane_off + c * 32, o);
          }
          tc::tmem_wait_st();
          if (need) { l *= f; m_used = mx; }
        }
      } else {
        m_used = mx;
      }
      const float mu = m_used == -INFINITY ? 0.f : m_used;
      float sum = 0.f;
      uint8_t* prow = sP + r * 128;
#pragma unroll
      for (int c8 = 0; c8 < 16; ++c8) {                   // 16 chunks of 8 keys (16 B)
        uint32_t pk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float p0 = tc::fast_exp2(x[c8 * 8 + 2 * e] - mu);
          const float p1 = tc::fast_exp2(x[c8 * 8 + 2 * e + 1] - mu);
          sum += p0 + p1;
          pk[e] = tc::pack_bf16(p0, p1);
        }
        const int blk = c8 >> 3, cc = c8 & 7;
        uint4* dst = reinterpret_cast<uint4*>(prow + blk * kTileBytes + ((cc ^ (r & 7)) << 4));
        *dst = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
      l += sum;
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(p_full);
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
      tc::tmem_ld32(tO + lane_off + c * 32, o);
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
    if (store) p.lse2[((long long)b * p.Hq + h) * p.M + qi] = m_used + log2f(l);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem);
  }
}

template <int D>
__global__ void __launch_bounds__(256, 1)
attn_score_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     TcParams p) {
  constexpr int KB = D / 64;
  constexpr int kStages = 3;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;                                   // KB blocks (the 128 keys, A operand)
  uint8_t* sQ = sK + KB * kTileBytes;                   // kStages x KB blocks
  float* sb = reinterpret_cast<float*>(sQ + kStages * KB * kTileBytes);   // [2][128] bias per query
  uint64_t* bars = reinterpret_cast<uint64_t*>(sb + 256);
  uint64_t* k_full = bars + 0;
  uint64_t* q_full = bars + 1;       // [3]
  uint64_t* q_empty = bars + 4;      // [3]
  uint64_t* s_full = bars + 7;       // [2]
  uint64_t* s_free = bars + 9;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int bgi = blockIdx.y;
  const int b = bgi / p.Hkv, gkv = bgi - b * p.Hkv;
  const long long bg = bgi;
  const bool resident = tile < p.n_res_tiles;
  int kstart, klen, k0 = 0;
  if (resident) {
    const int2 t = p.res_tiles[tile];
    kstart = t.x; klen = t.y;
  } else {
    k0 = (tile - p.n_res_tiles) * 128;
    kstart = p.S_tot + k0;
    klen = min(128, p.m - k0);
  }
  const int nqt = (p.m + 127) / 128;
  const int qt_begin = resident ? 0 : k0 / 128;
  const int per_head = nqt - qt_begin;
  const int n_items = p.G * per_head;

  if (threadIdx.x == 0) {
    tc::mbar_init(k_full, 1);
    for (int i = 0; i < kStages; ++i) { tc::mbar_init(q_full + i, 1); tc::mbar_init(q_empty + i, 1); }
    for (int i = 0; i < 2; ++i) { tc::mbar_init(s_full + i, 1); tc::mbar_init(s_free + i, 4); }
    tc::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tc::tma_prefetch(&tm_q); tc::tma_prefetch(&tm_k); }
  if (warp == 2) tc::tmem_alloc<256>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (tc::elect_one()) {
      const int krow = (int)(bg * (p.S_tot + p.M) + kstart);
      tc::mbar_expect_tx(k_full, KB * kTileBytes);
      for (int kb = 0; kb < KB; ++kb) tc::tma_load_2d(sK + kb * kTileBytes, &tm_k, k_full, kb * 64, krow);
      for (int i = 0; i < n_items; ++i) {
        const int st = i % kStages, u = i / kStages;
        if (i >= kStages) tc::mbar_wait(q_empty + st, (u - 1) & 1);
        const int hh = gkv * p.G + i / per_head;
        const int q0 = (qt_begin + i % per_head) * 128;
        const int qrow = (int)(((long long)b * p.Hq + hh) * p.M + q0);
        tc::mbar_expect_tx(q_full + st, KB * kTileBytes);
        for (int kb = 0; kb < KB; ++kb)
          tc::tma_load_2d(sQ + (st * KB + kb) * kTileBytes, &tm_q, q_full + st, kb * 64, qrow);
      }
    }
  } else if (warp == 1) {
    if (tc::elect_one()) {
      constexpr uint32_t idesc = tc::idesc_bf16_f32(128, 128, 0);
      const uint32_t aK = tc::smem_u32(sK), aQ = tc::smem_u32(sQ);
      tc::mbar_wait(k_full, 0);
      for (int i = 0; i < n_items; ++i) {
        const int st = i % kStages, s = i & 1;
        tc::mbar_wait(q_full + st, (i / kStages) & 1);
        if (i >= 2) tc::mbar_wait(s_free + s, ((i >> 1) - 1) & 1);
        tc::tc_fence_after();
        const uint32_t qb = aQ + st * KB * kTileBytes;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t da = tc::desc_kmajor_sw128(aK + (kk >> 2) * kTileBytes + (kk & 3) * 32);
          const uint64_t db = tc::desc_kmajor_sw128(qb + (kk >> 2) * kTileBytes + (kk & 3) * 32);
          tc::mma_bf16_ss(tmem + s * 128, da, db, idesc, kk > 0 ? 1u : 0u);
        }
        tc::mma_commit(s_full + s);
        tc::mma_commit(q_empty + st);
      }
    }
  } else if (warp >= 4) {
    const int r = threadIdx.x - 128;                      // key row = TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int key_idx = resident ? 0 : k0 + r;            // chunk-relative key index (chunk tiles)
    float best = 0.f, acc = 0.f;
    float x[128];
    for (int i = 0; i < n_items; ++i) {
      const int s = i & 1;
      const int hh = gkv * p.G + i / per_head;
      const int q0 = (qt_begin + i % per_head) * 128;
      {   // bias b_q = lse2_q - log2 w_q (+inf for queries past m)
        const int q = q0 + r;
        sb[s * 128 + r] = q < p.m ? p.lse2[((long long)b * p.Hq + hh) * p.M + q] - p.log2w[q] : INFINITY;
      }
      tc::named_bar_sync(1, 128);
      tc::mbar_wait(s_full + s, (i >> 1) & 1);
      tc::tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) tc::tmem_ld32(tmem + s * 128 + lane_off + c * 32, x + c * 32);
      tc::tmem_wait_ld();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(s_free + s);
      const float* bq = sb + s * 128;
      if (resident || q0 >= k0 + 128) {                    // no causal cut inside this block
#pragma unroll
        for (int c = 0; c < 128; ++c) acc += tc::fast_exp2(fmaf(x[c], p.scale_log2, -bq[c]));
      } else {
#pragma unroll
        for (int c = 0; c < 128; ++c) {
          const float e = tc::fast_exp2(fmaf(x[c], p.scale_log2, -bq[c]));
          acc += (q0 + c >= key_idx) ? e : 0.f;
        }
      }
      if ((i + 1) % per_head == 0) {                       // head finished: max over the group
        best = fmaxf(best, acc);
        acc = 0.f;
      }
    }
    if (r < klen) p.s[bg * (p.S_tot + p.m) + kstart + r] = best;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc<256>(tmem);
  }
}

size_t attn_fwd_tc_smem(int d) {
  const int KB = d / 64;
  return 1024 + (size_t)(KB + 2 + 2 * 2 * KB) * kTileBytes + 16 * 8 + 64;
}
size_t attn_score_tc_smem(int d) {
  const int KB = d / 64;
  return 1024 + (size_t)(KB + 3 * KB) * kTileBytes + 256 * 4 + 16 * 8 + 64;
}

void launch_attn_fwd_tc(const TcParams& p, const CUtensorMap& tq, const CUtensorMap& tk,
                        const CUtensorMap& tvs, const CUtensorMap& tvc, int d, cudaStream_t st) {
  dim3 grid((p.m + 127) / 128, p.Hq, p.B);
  const size_t smem = attn_fwd_tc_smem(d);
  if (d == 128) {
    cudaFuncSetAttribute(attn_fwd_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attn_fwd_tc_kernel<128><<<grid, 256, smem, st>>>(tq, tk, tvs, tvc, p);
  } else {
    cudaFuncSetAttribute(attn_fwd_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attn_fwd_tc_kernel<64><<<grid, 256, smem, st>>>(tq, tk, tvs, tvc, p);
  }
}

void launch_attn_score_tc(const TcParams& p, const CUtensorMap& tq, const CUtensorMap& tk, int d,
                          cudaStream_t st) {
  dim3 grid(p.n_res_tiles + (p.m + 127) / 128, p.B * p.Hkv);
  const size_t smem = attn_score_tc_smem(d);
  if (d == 128) {
    cudaFuncSetAttribute(attn_score_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attn_score_tc_kernel<128><<<grid, 256, smem, st>>>(tq, tk, p);
  } else {
    cudaFuncSetAttribute(attn_score_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attn_score_tc_kernel<64><<<grid, 256, smem, st>>>(tq, tk, p);
  }
}

}  // namespace cascade
