// k_decode.cu -- single-token step (Eq. 2) + its cascade update, bf16, ONE launch.
//
// Decode is HBM-bound (every cached K/V row is read once per step, ~4 flop/byte); the dot
// products still run on the tensor cores (tcgen05, M = 128 keys x N = 16 query columns) so the
// SIMT pipes are free for the per-key rotation and softmax.
//
// decode_fused_kernel: grid (nsplit, B*Hkv), one thread-block CLUSTER of nsplit CTAs per (b, g).
// Each CTA streams a contiguous range of the host's 128-slot key tiles (+ the new token's tile),
// rotates every raw key to its rank pe in shared memory, S^T = K_rot Q^T and
// O^T += V^T P^T in TMEM with an online softmax, and keeps every key's G log2-domain logits in
// TMEM (a compact column region, GM columns per tile).  Then, inside the same kernel:
//   1. cluster exchange (DSMEM) of each CTA's per-head (max, sum): every CTA knows the final
//      LSE of the G heads;
//   2. exact per-key mass s = w_0 * max_h exp2(logit_h - lse2_h) (Alg. 3 with m = 1: w_0 =
//      1 - gamma; max over the group; mean / median ablations) from the logits still in
//      TMEM -- no logits round trip through HBM -- written to s and folded into mu
//      (mu <- gamma * mu + s, IEEE double, never an FMA);
//   3. cluster rank 0 merges the CTAs' scaled partial O (DSMEM) into the bf16 output;
//   4. cluster rank 0 applies Alg. 2's single insertion: the (at most one) selection
//      on the folded mu (strict '>') and the (at most N+1) row moves, deepest sub-cache
//      first -- after a cluster barrier, so every CTA's fold is visible and every CTA's K/V
//      reads are done.
// The homogeneous head policy needs a reduction over the kv-heads of a sequence, i.e.
// across clusters: the fused kernel then only writes s, and decode_update_kernel folds, selects
// and moves after head_homogenize_kernel.
//
// Rotation precision (reading Q17): the oracle's key operand is the bf16 rounding of the exact R(pe) k
// (its float64 rotation rounded double -> float -> bf16; rope_prep computes exactly that).  The
// decode kernel rotates in fp32 on packed fp32x2 lanes (angle addition from the fp32 hi parts of
// double-float tables): error <= 3 * 2^-24 (|x1| + |x2|), so its bf16 rounding differs from the
// exact one for ~2e-5 of the elements (by one bf16 ulp of one coordinate).  With
// CASCADE_OPT_EXACT_DECODE_ROPE the kernel proves each rounding with an interval check and
// recomputes the unprovable pairs (~2e-3 of them) in double from the double-float tables -- exact
// operands, at ~+45 % decode time (the divergent fixups), so it is the parity mode, not the default.  (Rotating everything in
// float64 measured 1.21 vs 0.89 ms per configs[3] step: the DMUL / F2F issue of two warpgroups.)
#include "common.cuh"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <type_traits>
#include "tc_util.cuh"

namespace cascade {

namespace {
constexpr int kHiRows = 5;                                   // a-rows per tile: 128 consecutive pe span <= 5
constexpr int kLoRows = 32;                                  // pe = 32 a + b
constexpr int kLoStride = 64 * 8 + 16;                       // padded bytes per b-row (16-B aligned, bank spread)
constexpr int kKStages = 3;
constexpr int kTileBytes32K = 32768;                         // one 128 x 128 bf16 K or V tile
constexpr uint32_t kColLg = 64;                              // compact logits: GM columns per tile
constexpr uint32_t kTmemCols = 512;
#ifndef CASCADE_DEC_ROT_WG
#define CASCADE_DEC_ROT_WG 2
#endif
#ifndef CASCADE_DEC_PBUF
#define CASCADE_DEC_PBUF 2
#endif
constexpr int kPBuf = CASCADE_DEC_PBUF;                      // P^T buffers (2: softmax(j) overlaps PV(j-1))
// EXACT: the rotation proves every bf16 rounding and recomputes the unprovable pairs from the
// double-float tables, which needs the tables' lo parts in shared memory (a-rows of 1 KB, a second
// b-row table) and leaves room for two V stages; the fast variant stages hi parts only, three V stages.
template <bool EXACT> struct DecLayout {
  // rotation warpgroups: the exact variant's provable-rounding check and recomputation make the
  // rotation heavier, so it gets a third group (1.22 vs 1.35 ms per configs[3] step); the fast
  // variant measured the same with two and three (0.924 / 0.926 ms)
  static constexpr int kRotWG = EXACT ? 3 : CASCADE_DEC_ROT_WG;
  static constexpr int kThreads = 256 + 128 * kRotWG;
  static constexpr int kVStages = (EXACT || kPBuf == 2) ? 2 : 3;   // 227 KB: 3 V stages only with one P^T buffer
  static constexpr int kRowBytes = EXACT ? 1024 : 512;      // a-row: [64 float2 hi | 64 float2 lo] or hi only
  static constexpr int kARows = kHiRows * kRowBytes;        // a-rows per K stage
  static constexpr int kLoTables = EXACT ? 2 : 1;
  // sK | sV | sQ | sP | sA | sLo (| sLoL) | tile records | scalars + barriers; sO aliases sQ / sP
  // after the tiles
  static constexpr int max_tiles(int GM) { return (int)((kTmemCols - kColLg) / GM); }
  static constexpr size_t smem(int GM) {
    return (size_t)kKStages * kTileBytes32K + (size_t)kVStages * kTileBytes32K + 4096 + kPBuf * 4096 +
           (size_t)kKStages * kARows + (size_t)kLoTables * kLoRows * kLoStride + (size_t)max_tiles(GM) * 8 +
           4 * 8 * 4 + 40 * 4 + 64 + 24 * 8 + 1024;
  }
};
}  // namespace

size_t decode_fused_smem(int GM, bool exact) { return exact ? DecLayout<true>::smem(GM) : DecLayout<false>::smem(GM); }
int decode_fused_max_tiles(int GM) { return (int)((kTmemCols - kColLg) / GM); }

// Tensor-core decode, warp roles (DecLayout::kThreads = 256 + 128 kRotWG threads):
//   warp 0     producer: TMA of the raw K tile (SWIZZLE_128B) + the float64 cos/sin rows of the
//              tile's 32-position blocks (bulk copies) into a 3-stage K ring, freed by QK^T
//   warp 3     producer: TMA of the V tile into a 2-stage V ring, freed by PV
//   warp 1     MMA: S^T[128 keys x 16] = K_rot Q^T (two S^T buffers, so QK(j+1) runs during
//              softmax(j)), then O^T[128 d x 16] += V^T P^T
//   warp 2     TMEM allocator
//   warps 4-7  softmax: thread t = key t: logits (kept in TMEM), online softmax per head, P^T
//   warps 8+   kRotWG rotation warpgroups (the tile's 128 keys x 8 16-byte chunks of rotate-half
//              pairs dealt round-robin): rotate every raw key IN PLACE to its rank pe; they run up
//              to a full ring ahead of the softmax.  The rotation is the decode's issue-heaviest
//              stage; a third group measured no faster (0.926 vs 0.924 ms per configs[3] step).
// After the tiles, warps 4+ compute the masses and the fold; rank 0's softmax warps merge O
// and its warp 0 applies the insertion.
// Tile descriptor (int4, host): start slot, length, pe of key 0 (pe of key j = pe0 + j: the host
// splits a tile where a full ring wraps past its oldest slot).
// Optional per-CTA timeline (build with CASCADE_NVCC_EXTRA=-DCASCADE_DEC_TRACE; the default build
// has none of it): globaltimer at CTA start, after the prologue, after the last tile's softmax,
// after the mass / fold epilogue, at the end.  CASCADE_DEC_TRACE=n (env) dumps launch n.
#ifdef CASCADE_DEC_TRACE
__device__ unsigned long long* g_dec_trace = nullptr;
#define DEC_MARK(k)                                                                              \
  do {                                                                                            \
    if (g_dec_trace) {                                                                            \
      unsigned long long _t;                                                                      \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                                      \
      g_dec_trace[((long long)blockIdx.y * gridDim.x + blockIdx.x) * 8 + (k)] = _t;               \
    }                                                                                             \
  } while (0)
#else
#define DEC_MARK(k)
#endif

template <int GM, bool EXACT>
__global__ void __launch_bounds__(DecLayout<EXACT>::kThreads, 1) decode_fused_kernel(const __grid_constant__ CUtensorMap tm_k,
                                                              const __grid_constant__ CUtensorMap tm_v,
                                                              DecodeParams p, PlanDev pl, int32_t n_sel,
                                                              const int32_t* __restrict__ phase_begin,
                                                              int32_t n_phase, __nv_bfloat16* __restrict__ out) {
  constexpr int D = 128, HALF = 64;
  using Lay = DecLayout<EXACT>;
  constexpr int kVStages = Lay::kVStages, kRowBytes = Lay::kRowBytes, kRotWG = Lay::kRotWG;
  extern __shared__ __align__(1024) uint8_t dsm_raw[];
  uint8_t* dsm = dsm_raw + ((1024u - (tc::smem_u32(dsm_raw) & 1023u)) & 1023u);
  uint8_t* sK = dsm;                                        // kKStages x K tile (1 KB aligned for TMA)
  uint8_t* sV = sK + kKStages * kTileBytes32K;              // kVStages x V tile
  uint8_t* sQ = sV + kVStages * kTileBytes32K;              // [16 rows x 128 d] SW128 (2 x 2 KB)
  uint8_t* sP = sQ + 4096;                                  // 2 x [16 heads x 128 keys] SW128 (2 x 2 KB)
  uint8_t* sA = sP + kPBuf * 4096;                                  // kKStages x the tile's a-rows (cos/sin(32a theta))
  uint8_t* sLo = sA + kKStages * Lay::kARows;               // 32 x kLoStride: cos/sin(b theta_i), fp32 hi parts
  uint8_t* sLoL = sLo + (EXACT ? kLoRows * kLoStride : 0);  // (EXACT) their fp32 lo parts
  int2* sTile = reinterpret_cast<int2*>(sLoL + kLoRows * kLoStride);   // (start, len) of this CTA's tiles
  float (*sRed)[8] = reinterpret_cast<float (*)[8]>(sTile + Lay::max_tiles(GM));   // [4][8]
  float* sO = reinterpret_cast<float*>(sQ);                 // [GM][128] scaled partial O (after the tiles)
  float* sML = reinterpret_cast<float*>(sRed + 4);          // [0, 8) max, [8, 16) sum, [16, 24) lse2
  float* sCorr = sML + 24;                                  // [8]
  int* sRescale = reinterpret_cast<int*>(sCorr + 8);
  uint32_t* sTmem = reinterpret_cast<uint32_t*>(sRescale + 1);
  uint64_t* bars = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(sTmem + 1) + 7) & ~uintptr_t(7));
  uint64_t* kfull = bars + 0;       // [3]
  uint64_t* kempty = bars + 3;      // [3]
  uint64_t* rot_full = bars + 6;    // [3 stages]: every rotation warp arrives
  uint64_t* s_full = bars + 12;     // [2] per S^T buffer
  uint64_t* p_full = bars + 14;     // [2] per S^T buffer
  uint64_t* pv_done[2] = {bars + 16, bars + 23};   // PV of tiles j with j % 2 == i (sP buffer i)
  uint64_t* vfull = bars + 17;      // [kVStages <= 3]
  uint64_t* vempty = bars + 20;     // [kVStages <= 3]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int split = blockIdx.x, bg = blockIdx.y;
  const uint32_t crank = tc::cluster_ctarank();            // == split (cluster = the splits of bg)
  const int ns = gridDim.x;
  const int G = p.G;
  const int b = bg / p.Hkv, g = bg - b * p.Hkv;
  const int n_tiles = p.n_tiles + 1;                         // + the new-token tile
  const int per = (n_tiles + ns - 1) / ns;
  const int tbeg = split * per, tend = min(n_tiles, tbeg + per);
  const int nt = max(0, tend - tbeg);
  if (tid == 0) DEC_MARK(0);

  if (tid == 0) {
    for (int i = 0; i < kKStages; ++i) { tc::mbar_init(kfull + i, 1); tc::mbar_init(kempty + i, 1); }
    for (int i = 0; i < kVStages; ++i) { tc::mbar_init(vfull + i, 1); tc::mbar_init(vempty + i, 1); }
    for (int i = 0; i < kKStages; ++i) tc::mbar_init(rot_full + i, 4 * kRotWG);
    for (int i = 0; i < 2; ++i) { tc::mbar_init(s_full + i, 1); tc::mbar_init(p_full + i, 4); }
    tc::mbar_init(pv_done[0], 1);
    tc::mbar_init(pv_done[1], 1);
    tc::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tc::tma_prefetch(&tm_k); tc::tma_prefetch(&tm_v); }
  if (warp == 2) tc::tmem_alloc<kTmemCols>(sTmem);
  // group queries rotated to pe = n_cached (float64 rotation, Q17), bf16 (rows >= G zero);
  // cos/sin(b theta) rows
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
  for (int o = tid; o < kLoRows * HALF; o += blockDim.x) {     // tab_lo rows: [64 hi | 64 lo]
    const int rr = o / HALF, ii = o % HALF;
    *reinterpret_cast<float2*>(sLo + rr * kLoStride + ii * 8) = p.tab_lo[rr * 2 * HALF + ii];
    if (EXACT) *reinterpret_cast<float2*>(sLoL + rr * kLoStride + ii * 8) = p.tab_lo[rr * 2 * HALF + HALF + ii];
  }
  for (int o = tid; o < nt; o += blockDim.x) {              // the epilogue's tile records
    const int ti = tbeg + o;
    sTile[o] = ti < p.n_tiles ? make_int2(p.dec_tiles[ti].x, p.dec_tiles[ti].y) : make_int2(p.S_tot, 1);
  }
  for (int o = tid; o < kPBuf * 4096 / 16; o += blockDim.x) reinterpret_cast<uint4*>(sP)[o] = make_uint4(0u, 0u, 0u, 0u);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *sTmem, tO = tmem + 16;            // S^T buffers at columns 0 and 32
  if (tid == 0) DEC_MARK(1);

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
        const int s = j % kKStages;
        if (j >= kKStages) tc::mbar_wait(kempty + s, ((j / kKStages) - 1) & 1);
        int start, len, pe0;
        tile_info(tbeg + j, start, len, pe0);
        uint8_t* st = sK + s * kTileBytes32K;
        const int a0 = pe0 >> 5, nA = ((pe0 + len - 1) >> 5) - a0 + 1;
        const uint32_t bytes = (start < p.S_tot ? 32768u : 0u) + (uint32_t)nA * kRowBytes;
        tc::mbar_expect_tx(kfull + s, bytes);
        if (start < p.S_tot) {
          const int row = (int)((long long)bg * p.S_tot + start);
          for (int kb = 0; kb < 2; ++kb) tc::tma_load_2d(st + kb * 16384, &tm_k, kfull + s, kb * 64, row);
          // the epilogue folds this tile's mu: pull it into L2 now (off the HBM-latency tail)
          // (bulk prefetch: 16-B aligned start and size, so the range is trimmed to whole pairs)
          const long long x0 = ((long long)bg * p.S_tot + start + 1) & ~1LL;
          const long long x1 = ((long long)bg * p.S_tot + start + len) & ~1LL;
          if (p.update && x1 > x0) tc::bulk_prefetch_l2(p.mu + x0, (uint32_t)(x1 - x0) * 8u);
        }
        for (int r = 0; r < nA; ++r)
          tc::bulk_load(sA + s * Lay::kARows + r * kRowBytes, p.tab_hi + (long long)(a0 + r) * 2 * HALF, kRowBytes,
                        kfull + s);
      }
    }
  } else if (warp == 3) {
    if (tc::elect_one()) {
      for (int j = 0; j < nt; ++j) {              // V tiles (the new token's V is written by the rotation warps)
        const int s = j % kVStages;
        if (j >= kVStages) tc::mbar_wait(vempty + s, ((j / kVStages) - 1) & 1);
        int start, len, pe0;
        tile_info(tbeg + j, start, len, pe0);
        uint8_t* st = sV + s * kTileBytes32K;
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
        const int s = j % kKStages;
        const uint32_t st = tc::smem_u32(sK + s * kTileBytes32K);
        tc::mbar_wait(rot_full + s, (j / kKStages) & 1);           // every rotated chunk in place
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
        const int s = j % kVStages;
        const uint32_t st = tc::smem_u32(sV + s * kTileBytes32K);
        tc::mbar_wait(p_full + (j & 1), (j >> 1) & 1);       // P^T written (and O^T rescaled)
        tc::mbar_wait(vfull + s, (j / kVStages) & 1);
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t da = tc::desc_mnmajor_sw128(st + kk * 2048, 16384);
          const uint64_t db = tc::desc_kmajor_sw128(aP + (kPBuf == 2 ? (j & 1) * 4096 : 0) + (kk >> 2) * 2048 + (kk & 3) * 32);
          tc::mma_bf16_ss(tO, da, db, idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit(pv_done[j & 1]);
        tc::mma_commit(vempty + s);
      }
    }
  } else if (warp >= 8) {
    // ---------------- rotation warpgroups ----------------
    const int t = (tid - 256) & 127;                         // key row of the tile (fixed per thread)
    const int c0 = (tid - 256) >> 7;                         // chunks c0, c0 + kRotWG, ... (< 8)
    for (int j = 0; j < nt; ++j) {
      const int s = j % kKStages;
      uint8_t* st = sK + s * kTileBytes32K;
      int start, len, pe0;
      tile_info(tbeg + j, start, len, pe0);
      const bool valid = t < len;
      const int pe = pe0 + t;
      tc::mbar_wait(kfull + s, (j / kKStages) & 1);
      if (start < p.S_tot) {
        // ---- rotate row t in place: pairs (i, i + 64) live at the same swizzled offset of the
        //      two 64-column blocks.  Fast path in fp32: cos/sin((32a + b) theta_i) by angle
        //      addition from fp32 tables (a-rows staged per tile, b-rows resident); its error is
        //      below 16 * 2^-24 * (|x1| + |x2|) (table rounding, two products, two roundings), so
        //      its bf16 rounding equals that of the exact rotation unless the fp32 value lies that
        //      close to a bf16 rounding midpoint -- then (~2e-4 of the elements) the pair is
        //      recomputed exactly as rope_prep does it: fp64 table, double products, double ->
        //      float -> bf16 (reading Q17).
        const int hr = (pe >> 5) - (pe0 >> 5);
        const float2* hi = reinterpret_cast<const float2*>(sA + s * Lay::kARows + (valid ? hr : 0) * kRowBytes);
        const float2* lo = reinterpret_cast<const float2*>(sLo + (pe & 31) * kLoStride);
        const float2* lo_l = reinterpret_cast<const float2*>(sLoL + (pe & 31) * kLoStride);
#pragma unroll 1
        for (int c = c0; c < 8; c += kRotWG) {
          const int off = t * 128 + ((c ^ (t & 7)) << 4);
          uint4* pa = reinterpret_cast<uint4*>(st + off);
          uint4* pb = reinterpret_cast<uint4*>(st + 16384 + off);
          const uint4 ua = *pa, ub = *pb;
          const uint32_t wa[4] = {ua.x, ua.y, ua.z, ua.w}, wb[4] = {ub.x, ub.y, ub.z, ub.w};
          uint32_t oa[4], ob[4];
#pragma unroll
          for (int e2 = 0; e2 < 4; ++e2) {          // pairs i0, i0 + 1 as packed fp32x2 lanes
            const int i0 = c * 8 + 2 * e2;
            const float4 hh = *reinterpret_cast<const float4*>(hi + i0);   // c_i, s_i, c_i+1, s_i+1
            const float4 ll = *reinterpret_cast<const float4*>(lo + i0);
            const float2 cA = make_float2(hh.x, hh.z), sA = make_float2(hh.y, hh.w);
            const float2 cB = make_float2(ll.x, ll.z), sB = make_float2(ll.y, ll.w);
            const float2 cs = __ffma2_rn(cA, cB, __fmul2_rn(sA, make_float2(-sB.x, -sB.y)));   // cos(A + B)
            const float2 sn = __ffma2_rn(sA, cB, __fmul2_rn(cA, sB));                         // sin(A + B)
            const float2 x1 = make_float2(__uint_as_float(wa[e2] << 16), __uint_as_float(wa[e2] & 0xffff0000u));
            const float2 x2 = make_float2(__uint_as_float(wb[e2] << 16), __uint_as_float(wb[e2] & 0xffff0000u));
            const float2 y1 = __ffma2_rn(x1, cs, __fmul2_rn(make_float2(-x2.x, -x2.y), sn));  // x1 c - x2 s
            const float2 y2 = __ffma2_rn(x2, cs, __fmul2_rn(x1, sn));                         // x2 c + x1 s
            // |y - exact| <= 3 * 2^-24 (|x1| + |x2|) (four table entries at half an ulp, |cos|,
            // |sin| <= 1, one product and one fma rounding).  With delta = 4e-7 (|x1| + |x2|)
            // (> that bound + half an ulp of y), [y - delta, y + delta] holds the exact value, so
            // when both ends round to the same bf16 so does the exact rotation (rounding is
            // monotonic) and that bf16 is the result; otherwise the pair is recomputed exactly.
            uint32_t r1, r2;
            bool fix = false;
            if (EXACT) {
              const float2 dl = __fmul2_rn(__fadd2_rn(make_float2(fabsf(x1.x), fabsf(x1.y)),
                                                      make_float2(fabsf(x2.x), fabsf(x2.y))),
                                           make_float2(4e-7f, 4e-7f));
              const float2 nd = make_float2(-dl.x, -dl.y);
              const float2 y1l = __fadd2_rn(y1, nd), y1h = __fadd2_rn(y1, dl);
              const float2 y2l = __fadd2_rn(y2, nd), y2h = __fadd2_rn(y2, dl);
              r1 = tc::pack_bf16(y1l.x, y1l.y);
              r2 = tc::pack_bf16(y2l.x, y2l.y);
              fix = valid && (r1 != tc::pack_bf16(y1h.x, y1h.y) || r2 != tc::pack_bf16(y2h.x, y2h.y));
            } else {                                 // fast variant: the fp32 rotation's own rounding
              r1 = tc::pack_bf16(y1.x, y1.y);
              r2 = tc::pack_bf16(y2.x, y2.y);
            }
            if (EXACT && fix) {
              // exact: cos / sin from the double-float tables (hi + lo) by angle addition in
              // double, then rope_prep's arithmetic (double products, double -> float -> bf16)
              float o1[2], o2[2];
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                const int i = i0 + u;
                const float2 h2 = hi[i], h2l = hi[HALF + i], l2 = lo[i], l2l = lo_l[i];
                const double ca = (double)h2.x + (double)h2l.x, sa = (double)h2.y + (double)h2l.y;
                const double cb = (double)l2.x + (double)l2l.x, sb = (double)l2.y + (double)l2l.y;
                const double c64 = ca * cb - sa * sb, s64 = sa * cb + ca * sb;
                const double d1 = u ? x1.y : x1.x, d2 = u ? x2.y : x2.x;
                o1[u] = __double2float_rn(__dsub_rn(__dmul_rn(d1, c64), __dmul_rn(d2, s64)));
                o2[u] = __double2float_rn(__dadd_rn(__dmul_rn(d2, c64), __dmul_rn(d1, s64)));
              }
              r1 = tc::pack_bf16(o1[0], o1[1]);
              r2 = tc::pack_bf16(o2[0], o2[1]);
            }
            oa[e2] = r1;
            ob[e2] = r2;
          }
          *pa = make_uint4(oa[0], oa[1], oa[2], oa[3]);
          *pb = make_uint4(ob[0], ob[1], ob[2], ob[3]);
        }
      } else {
        // ---- the new token: key row 0 from the input, rotated to n_cached; rows >= 1 zero;
        //      its V row goes to the V stage once that is free ----
        const int sv_i = j % kVStages;
        tc::mbar_wait(vfull + sv_i, (j / kVStages) & 1);
        uint8_t* sv = sV + sv_i * kTileBytes32K;
        const int off_base = t * 128;
        for (int c = c0; c < 8; c += kRotWG) {
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
      if (lane == 0) tc::mbar_arrive(rot_full + s);
    }
  } else if (warp >= 4) {
    // ---------------- softmax warpgroup ----------------
    const int t = tid - 128;                                 // key = TMEM lane
    const int w4 = warp & 3;
    const uint32_t lane_off = (uint32_t)(w4 * 32) << 16;
    float m_run[GM], l_part[GM];
#pragma unroll
    for (int h = 0; h < GM; ++h) { m_run[h] = -INFINITY; l_part[h] = 0.f; }
    for (int j = 0; j < nt; ++j) {
      int start, len, pe0;
      tile_info(tbeg + j, start, len, pe0);
      const bool valid = t < len;
      // ---- logits (kept in TMEM for the mass), block max per head, P^T ----
      tc::mbar_wait(s_full + (j & 1), (j >> 1) & 1);
      tc::tc_fence_after();
      float sv[16];
      tc::tmem_ld16(tmem + (j & 1) * 32 + lane_off, sv);
      tc::tmem_wait_ld();
      float lg[GM];
      uint32_t lgb[GM];
#pragma unroll
      for (int h = 0; h < GM; ++h) {
        lg[h] = (valid && h < G) ? sv[h] * p.scale_log2 : -INFINITY;
        lgb[h] = __float_as_uint(lg[h]);
      }
      tc::tmem_st_n<GM>(tmem + lane_off + kColLg + (uint32_t)(GM * j), lgb);
#pragma unroll
      for (int h = 0; h < GM; ++h) {
        float v = lg[h];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) sRed[w4][h] = v;
      }
      tc::named_bar_sync(1, 128);
      if (t == 0) {
        int any = 0;
#pragma unroll
        for (int h = 0; h < GM; ++h) {
          const float mt = fmaxf(fmaxf(sRed[0][h], sRed[1][h]), fmaxf(sRed[2][h], sRed[3][h]));
          const float mn = fmaxf(m_run[h], mt);
          const float cr = (m_run[h] == -INFINITY) ? 0.f : exp2f(m_run[h] - mn);
          sCorr[h] = cr;
          any |= (j > 0 && m_run[h] != -INFINITY && cr != 1.f);
          sRed[0][h] = mn;
        }
        *sRescale = any;
      }
      tc::named_bar_sync(1, 128);
      // sP[j % 2] is free once PV(j-2) is done; a rescale of O^T needs every PV < j (PV(j-1)
      // done: tcgen05 MMAs of one thread complete in order).  One barrier per buffer, so a
      // parity wait is never ambiguous (PV(j) cannot complete before this P is written).
      if (*sRescale || kPBuf == 1) {
        if (j >= 1) tc::mbar_wait(pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
      } else if (j >= 2) {
        tc::mbar_wait(pv_done[j & 1], ((j - 2) >> 1) & 1);
      }
      tc::tc_fence_after();
#pragma unroll
      for (int h = 0; h < GM; ++h) {
        const float mn = sRed[0][h];
        const float cr = sCorr[h];
        m_run[h] = mn;
        const float pv = (valid && h < G) ? exp2f(lg[h] - mn) : 0.f;
        l_part[h] = l_part[h] * cr + pv;
        const int blk = t >> 6, kc = t & 63;
        *reinterpret_cast<__nv_bfloat16*>(sP + (kPBuf == 2 ? (j & 1) * 4096 : 0) + blk * 2048 + h * 128 + ((((kc >> 3) ^ (h & 7))) << 4) + (kc & 7) * 2) =
            __float2bfloat16_rn(pv);
      }
      if (*sRescale) {                                       // O^T column h *= corr_h (lane = d)
        float ov[16];
        tc::tmem_ld16(tO + lane_off, ov);
        tc::tmem_wait_ld();
#pragma unroll
        for (int h = 0; h < GM; ++h) ov[h] *= sCorr[h];
        tc::tmem_st16(tO + lane_off, reinterpret_cast<const uint32_t*>(ov));
        tc::tmem_wait_st();
      }
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      tc::named_bar_sync(1, 128);                            // sRed / sCorr reads done
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(p_full + (j & 1));
    }
    // ---- this CTA's per-head (max, sum) ----
#pragma unroll
    for (int h = 0; h < GM; ++h) {
      float v = l_part[h];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) sRed[w4][h] = v;
    }
    if (nt > 1) tc::mbar_wait(pv_done[(nt - 2) & 1], ((nt - 2) >> 1) & 1);   // every phase observed
    if (nt > 0) tc::mbar_wait(pv_done[(nt - 1) & 1], ((nt - 1) >> 1) & 1);   // O^T holds every tile
    if (t == 0) DEC_MARK(2);
    tc::tmem_wait_st();
    tc::named_bar_sync(1, 128);
    if (t < GM) {
      sML[t] = m_run[t];
      sML[8 + t] = sRed[0][t] + sRed[1][t] + sRed[2][t] + sRed[3][t];
    }
  }
  // ======== cluster exchange #1: every CTA's (max, sum) per head ========
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();
  tc::tc_fence_after();
  if (tid < GM) {                                            // final log2-domain LSE of head tid
    float mr[8], lr[8];                                      // every CTA's (max, sum): loads first
#pragma unroll
    for (int r = 0; r < 8; ++r)
      if (r < ns) { mr[r] = tc::ld_cluster_f32(sML + tid, (uint32_t)r); lr[r] = tc::ld_cluster_f32(sML + 8 + tid, (uint32_t)r); }
    float M = -INFINITY;
#pragma unroll
    for (int r = 0; r < 8; ++r)
      if (r < ns) M = fmaxf(M, mr[r]);
    float L = 0.f;
#pragma unroll
    for (int r = 0; r < 8; ++r)
      if (r < ns && mr[r] != -INFINITY) L += lr[r] * exp2f(mr[r] - M);
    sML[16 + tid] = M + log2f(L);
    sCorr[tid] = (sML[tid] == -INFINITY) ? 0.f : exp2f(sML[tid] - M) / L;   // this CTA's O weight
  }
  __syncthreads();
  if (tid == 0) DEC_MARK(5);
  {
    // every warp shares the tiles now (TMEM lanes 32 (warp % 4) .. + 31 are each warp's own)
    constexpr int kWG = 2 + kRotWG;
    const int wg = warp >> 2;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int t = (warp & 3) * 32 + lane;                    // key (or d) = TMEM lane
    if (wg == 1) {                                           // scaled partial O^T -> sO (own smem)
      float ov[16];
      tc::tmem_ld16(tO + lane_off, ov);
      tc::tmem_wait_ld();
#pragma unroll
      for (int h = 0; h < GM; ++h) sO[h * 128 + t] = ov[h] * sCorr[h];
    }
    // ---- exact per-key mass (Alg. 3, m = 1) + EMA fold, from the logits in TMEM ----
    float lse[GM];
#pragma unroll
    for (int h = 0; h < GM; ++h) lse[h] = sML[16 + h];
    double* mu = p.mu + (long long)bg * p.S_tot;
    float* s_out = p.s + (long long)bg * (p.S_tot + 1);
    // kU tiles per round: every TMEM load and mu load of the round is issued before the first
    // use (tile records in shared memory, mu prefetched into L2 with its K tile), so the tail pays
    // one L2 round trip per round
    constexpr int kU = GM >= 8 ? 4 : GM >= 4 ? 6 : 8;
    for (int j0 = wg; j0 < nt; j0 += kWG * kU) {
      uint32_t lgb[kU][GM];
      double m0[kU];
      int xs[kU];
      bool vk[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int j = j0 + kWG * u;
        int start = 0, len = 0;
        if (j < nt) {
          const int2 tr = sTile[j];
          start = tr.x; len = tr.y;
          tc::tmem_ld_n<GM>(tmem + lane_off + kColLg + (uint32_t)(GM * j), lgb[u]);
        }
        vk[u] = j < nt && t < len;
        xs[u] = start + t;
        m0[u] = (vk[u] && xs[u] < p.S_tot && p.update) ? mu[xs[u]] : 0.0;
      }
      tc::tmem_wait_ld();
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (!vk[u]) continue;
        float best = 0.f;
        if (p.head_reduce == 0) {
#pragma unroll
          for (int h = 0; h < GM; ++h)
            if (h < G) best = fmaxf(best, exp2f(__uint_as_float(lgb[u][h]) - lse[h]));
        } else {                                             // mean / median ablations
          float hv[GM];
#pragma unroll
          for (int h = 0; h < GM; ++h) hv[h] = h < G ? exp2f(__uint_as_float(lgb[u][h]) - lse[h]) : 0.f;
          if (p.heads_out)                                   // homogeneous + median: every head's mass
            for (int h = 0; h < G; ++h)
              p.heads_out[((long long)b * p.Hq + g * G + h) * p.heads_ld + xs[u]] = p.w0 * hv[h];
          best = group_reduce_ablation(hv, G, p.head_reduce);
        }
        const float sv = p.w0 * best;
        s_out[xs[u]] = sv;
        if (xs[u] < p.S_tot && p.update) mu[xs[u]] = __dadd_rn(__dmul_rn(p.decay, m0[u]), (double)sv);
      }
    }
  }
  if (tid == 128) DEC_MARK(3);
  // ======== cluster exchange #2: every fold and every s visible; partial O staged ========
  __threadfence();
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();
  tc::tc_fence_after();
  if (crank == 0) {
    if (warp >= 4 && warp < 8) {                             // O = sum over the cluster's CTAs
      const int d = tid - 128;
      for (int h = 0; h < G; ++h) {
        float o = 0.f;
        for (int r = 0; r < ns; ++r) o += tc::ld_cluster_f32(sO + h * 128 + d, (uint32_t)r);
        out[((long long)b * p.Hq + g * G + h) * D + d] = __float2bfloat16_rn(o);
      }
    }
  }
  // ======== #3: peers keep their shared memory until rank 0 has read it; then they may exit
  //          while rank 0 applies the insertion (it needs only global memory: every CTA's fold
  //          is visible since #2) ========
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();
  if (crank == 0 && warp == 0 && p.update) {
      // ---- Alg. 2's single insertion: selections (depth order), then moves deepest first ----
      double* mu = p.mu + (long long)bg * p.S_tot;
      const float* s_out = p.s + (long long)bg * (p.S_tot + 1);
      int32_t* res = pl.resolved + (long long)bg * pl.sel_cap;
      if (lane == 0) {
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
      // moves in phase order (deepest sub-cache first), kMB per round: every source of a round is
      // read before any of its destinations is written, rounds in order.  A move's destination
      // is only ever the source of an EARLIER move (the evictee it carried down), so
      // batching keeps the one-at-a-time semantics with one load round trip per round instead of
      // one per move.
      constexpr int NV = D * 2 / 16;                         // 16-B vectors per K (or V) row
      constexpr int kMB = 6;
      const int e_end = phase_begin[n_phase];
      for (int e0 = phase_begin[0]; e0 < e_end; e0 += kMB) {
        uint4 row[kMB];
        int32_t dsts[kMB];
        double mu_new = 0.0;
        int64_t org = 0;
#pragma unroll
        for (int u = 0; u < kMB; ++u) {
          const int e = e0 + u;
          dsts[u] = -1;
          if (e >= e_end) continue;
          const int32_t dst = pl.mov[2 * e];
          int32_t src = pl.mov[2 * e + 1];
          src = src >= 0 ? src : res[-src - 1];
          if (src == dst) continue;
          dsts[u] = dst;
          const __nv_bfloat16* rs;                           // lanes < NV: K, the rest: V
          if (src < p.S_tot) {
            rs = (lane < NV ? p.k_raw_mut : p.v_mut) + ((long long)bg * p.S_tot + src) * D;
            if (lane == u) { mu_new = mu[src]; org = p.origin[(long long)bg * p.S_tot + src]; }
          } else {
            rs = (lane < NV ? p.k_new : p.v_new) + (long long)bg * D;
            if (lane == u) { mu_new = (double)s_out[src]; org = p.t0; }
          }
          row[u] = reinterpret_cast<const uint4*>(rs)[lane & (NV - 1)];
        }
        __syncwarp();                                        // every read of the round done
#pragma unroll
        for (int u = 0; u < kMB; ++u) {
          if (dsts[u] < 0) continue;
          __nv_bfloat16* rd = (lane < NV ? p.k_raw_mut : p.v_mut) + ((long long)bg * p.S_tot + dsts[u]) * D;
          reinterpret_cast<uint4*>(rd)[lane & (NV - 1)] = row[u];
          if (lane == u) { mu[dsts[u]] = mu_new; p.origin[(long long)bg * p.S_tot + dsts[u]] = org; }
        }
        __syncwarp();
      }
  }
  if (tid == 0) DEC_MARK(4);
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc<kTmemCols>(tmem);
  }
}

// Stage 2 of the homogeneous head policy, one CTA per (b, g): s already holds the
// per-sequence reduction (head_homogenize_kernel); fold it into mu, then the selections and
// moves of the single insertion.
template <int D>
__global__ void __launch_bounds__(256) decode_update_kernel(DecodeParams p, PlanDev pl, int32_t n_sel,
                                                            const int32_t* __restrict__ phase_begin,
                                                            int32_t n_phase) {
  const int bg = blockIdx.x, tid = threadIdx.x;
  double* mu = p.mu + (long long)bg * p.S_tot;
  float* s_out = p.s + (long long)bg * (p.S_tot + 1);
  for (int run = 0; run <= p.N; ++run) {
    const int beg = run == 0 ? 0 : p.alpha + (run - 1) * p.c;
    const int len = run == 0 ? p.sink_pre : p.counts[run - 1];
    for (int o = tid; o < len; o += blockDim.x)
      mu[beg + o] = __dadd_rn(__dmul_rn(p.decay, mu[beg + o]), (double)s_out[beg + o]);
  }
  __syncthreads();
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
        const uint4 kv = reinterpret_cast<const uint4*>(ks)[tid & (NV - 1)];
        const uint4 vv = reinterpret_cast<const uint4*>(vs)[tid & (NV - 1)];
        __syncwarp();
        if (tid < NV) reinterpret_cast<uint4*>(kd)[tid] = kv;
        else reinterpret_cast<uint4*>(vd)[tid - NV] = vv;
        if (tid == 0) { mu[dst] = mu_new; p.origin[(long long)bg * p.S_tot + dst] = org; }
        __syncwarp();
      }
    }
  }
}

int decode_gm(int G) { return G <= 1 ? 1 : G <= 2 ? 2 : G <= 4 ? 4 : 8; }

size_t decode_nsplit(const DecodeParams& p) {
  // splits per (b, g) = cluster size: minimise (waves of 1-CTA-per-SM CTAs) x (tiles per CTA +
  // ~4 tiles of per-CTA pipeline fill / epilogue), subject to every tile's logits fitting in TMEM;
  // clusters of 2 tile the 148 SMs exactly, clusters of 4 strand 16 of them (B300_MICROARCH.md)
  const int GM = decode_gm(p.G);
  const int tiles = p.n_tiles + 1, cap = decode_fused_max_tiles(GM);
  const int bgs = p.B * p.Hkv;
  int best = 0;
  double best_cost = 1e300;
  for (int ns : {1, 2, 4, 8}) {
    const int per = (tiles + ns - 1) / ns;
    if (per > cap) continue;
    const double sms = ns <= 2 ? 148.0 : ns == 4 ? 132.0 : 128.0;
    const double cost = std::ceil((double)bgs * ns / sms) * (per + 4.0);
    if (cost < best_cost) { best_cost = cost; best = ns; }
  }
  return (size_t)best;            // 0: the cache is too large for the in-TMEM logits
}

template <int GM, bool EXACT>
cudaError_t launch_fused(const DecodeParams& p, const PlanDev& pl, int32_t n_sel, const int32_t* phase_begin_dev,
                         int32_t n_phase, __nv_bfloat16* out, const CUtensorMap& tk, const CUtensorMap& tv,
                         cudaStream_t st) {
  const size_t smem = DecLayout<EXACT>::smem(GM);
  auto kern = decode_fused_kernel<GM, EXACT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.nsplit, p.B * p.Hkv);
  cfg.blockDim = dim3(DecLayout<EXACT>::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.nsplit;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#ifdef CASCADE_DEC_TRACE
  static unsigned long long* trace = nullptr;
  static int trace_at = -1, calls = 0;
  const size_t ctas = (size_t)p.nsplit * p.B * p.Hkv;
  if (trace_at < 0) {
    const char* ev = std::getenv("CASCADE_DEC_TRACE");
    trace_at = ev ? std::atoi(ev) : 0;
    if (trace_at > 0) {
      cudaMalloc(&trace, ctas * 8 * 8);
      cudaMemcpyToSymbol(g_dec_trace, &trace, sizeof(trace));
    }
  }
#endif
  const cudaError_t rc = cudaLaunchKernelEx(&cfg, kern, tk, tv, p, pl, n_sel, phase_begin_dev, n_phase, out);
#ifdef CASCADE_DEC_TRACE
  if (trace_at > 0 && ++calls == trace_at) {
    std::vector<unsigned long long> h(ctas * 8);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, t1 = 0;
    for (size_t c = 0; c < ctas; ++c) { t0 = std::min(t0, h[c * 8]); t1 = std::max(t1, h[c * 8 + 4]); }
    double pro = 0, tiles = 0, lse = 0, epi = 0, fin = 0;
    for (size_t c = 0; c < ctas; ++c) {
      pro += h[c * 8 + 1] - h[c * 8]; tiles += h[c * 8 + 2] - h[c * 8 + 1];
      lse += h[c * 8 + 5] - h[c * 8 + 2]; epi += h[c * 8 + 3] - h[c * 8 + 5]; fin += h[c * 8 + 4] - h[c * 8 + 3];
    }
    std::fprintf(stderr, "decode trace: %zu CTAs, span %.1f us; per CTA avg: prologue %.2f us, tiles %.2f us, "
                 "cluster wait + LSE %.2f us, mass+fold %.2f us, exchange+insert %.2f us\n", ctas, (t1 - t0) / 1e3,
                 pro / ctas / 1e3, tiles / ctas / 1e3, lse / ctas / 1e3, epi / ctas / 1e3, fin / ctas / 1e3);
    for (size_t c = 0; c < ctas; c += ctas / 16)
      std::fprintf(stderr, "  cta %zu start %.1f tiles_end %.1f end %.1f us\n", c, (h[c * 8] - t0) / 1e3,
                   (h[c * 8 + 2] - t0) / 1e3, (h[c * 8 + 4] - t0) / 1e3);
  }
#endif
  return rc;
}

cudaError_t launch_decode_fused(const DecodeParams& p, const PlanDev& pl, int32_t n_sel,
                                const int32_t* phase_begin_dev, int32_t n_phase, __nv_bfloat16* out,
                                const CUtensorMap& tk, const CUtensorMap& tv, cudaStream_t st) {
  const int GM = decode_gm(p.G);
  auto go = [&](auto exact) {
    constexpr bool E = decltype(exact)::value;
    if (GM == 1) return launch_fused<1, E>(p, pl, n_sel, phase_begin_dev, n_phase, out, tk, tv, st);
    if (GM == 2) return launch_fused<2, E>(p, pl, n_sel, phase_begin_dev, n_phase, out, tk, tv, st);
    if (GM == 4) return launch_fused<4, E>(p, pl, n_sel, phase_begin_dev, n_phase, out, tk, tv, st);
    return launch_fused<8, E>(p, pl, n_sel, phase_begin_dev, n_phase, out, tk, tv, st);
  };
  return p.exact_rope ? go(std::true_type{}) : go(std::false_type{});
}

cudaError_t launch_decode_commit(const DecodeParams& p, const PlanDev& pl, int32_t n_sel,
                                 const int32_t* phase_begin_dev, int32_t n_phase, cudaStream_t st) {
  decode_update_kernel<128><<<p.B * p.Hkv, 256, 0, st>>>(p, pl, n_sel, phase_begin_dev, n_phase);
  return cudaGetLastError();
}

}  // namespace cascade
