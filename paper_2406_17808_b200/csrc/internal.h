// internal.h -- shared between the host control plane and the kernels (library-private).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../include/cascade.h"

namespace cascade {

// Per-call geometry of one layer's cascades, passed by value to every kernel.
// "pre" = state before the chunk (what attention sees and what the fold uses).
struct Geometry {
  int32_t B, Hq, Hkv, G, d;
  int32_t alpha, N, c, S_tot;           // S_tot = alpha + N*c
  int32_t m;                            // chunk length
  int32_t ldc;                          // row capacity of chunk-space scratch (max_stride)
  int64_t t0;                           // stream index of chunk row 0
  int32_t sink_pre;                     // sink residents before the chunk
  int32_t n_cached;                     // residents before the chunk
  int32_t counts_pre[CASCADE_MAX_LEVELS];
  int32_t xi_pre[CASCADE_MAX_LEVELS];
  int32_t base_pre[CASCADE_MAX_LEVELS]; // pe of the oldest token of sub-cache i (logical order)
  float scale;                          // softmax scale
  float scale_log2;                     // scale * log2(e)
  double decay;                         // g = gamma^m
  int32_t head_reduce;                  // GQA head reduction of s: 0 max; ablations 1 mean, 2 median
  int32_t homogeneous;                  // head policy: 0 independent, 1 homogeneous
};

// pe of a pre-chunk resident flat slot x (-1 if empty).  Closed form of the logical
// order [sinks; C_N oldest..newest; ...; C_1].
__host__ __device__ inline int32_t slot_pe(const Geometry& g, int32_t x) {
  if (x < g.alpha) return x < g.sink_pre ? x : -1;
  int32_t rel = x - g.alpha;
  int32_t i = rel / g.c;               // 0-based level
  int32_t s = rel - i * g.c;
  int32_t cnt = g.counts_pre[i];
  if (s >= cnt) return -1;
  int32_t rank = (cnt == g.c) ? ((s - g.xi_pre[i] + g.c) % g.c) : s;
  return g.base_pre[i] + rank;
}

struct Workspace;  // device carve (host side)

// Schedule of one chunk, in device memory (int32):
//   sel[3*k + {0,1,2}] = {slot, cand_ref, inc_ref}       k < n_sel
//   sel_order[]        = select indices sorted by dependency depth
//   mov[2*e + {0,1}]   = {dst_slot, ref}                 grouped by phase
// A ref >= 0 is a concrete source: flat slot (< S_tot, pre-chunk occupant) or
// chunk row (S_tot + r).  A ref < 0 is -(k+1): the winner of select k.
struct PlanDev {
  const int32_t* sel;
  const int32_t* sel_order;
  const int32_t* mov;
  int32_t* resolved;        // [B*Hkv][sel_cap]
  int32_t sel_cap;
};

template <typename T>
struct StateDev {
  T* k_raw;        // [B*Hkv][S_tot][d]
  T* v;            // [B*Hkv][S_tot][d]
  double* mu;      // [B*Hkv][S_tot]
  int64_t* origin; // [B*Hkv][S_tot]
  const T* k_in;   // [B][m][Hkv][d] this chunk's keys (pre-RoPE) and values (maintenance sources)
  const T* v_in;
};

// ---- launchers (defined in the .cu files) --------------------------------
template <typename T>
void launch_rope_prep(const Geometry& g, const T* q, const T* k, const T* v, const T* k_raw_state,
                      const double2* rope_tab, const float2* rope_tab_f, T* q_rot, T* k_rot, T* v_chunk, cudaStream_t st);

template <typename T>
void launch_attn_fwd_simt(const Geometry& g, const T* q_rot, const T* k_rot, const T* v_state,
                          const T* v_chunk, T* out, float* lse, cudaStream_t st);

template <typename T>
void launch_attn_score_simt(const Geometry& g, const T* q_rot, const T* k_rot, const float* lse,
                            const float* w, float* s, float* heads_out, int heads_ld, cudaStream_t st);


void launch_select_resolve(const Geometry& g, const PlanDev& p, int32_t begin, int32_t end,
                           const double* mu, const float* s, cudaStream_t st);

// One cooperative maintenance launch per chunk (k_maint.cu, maint_coop_kernel).
struct MaintItems {
  const int4* staged;         // [n_staged] {dst, ref, cand, inc}: moves reading a resident slot,
  int32_t n_staged;           //   in phase order (C_N .. C_1, sinks); cand/inc when ref < 0
  const int4* chunk;          // [n_chunk] moves that read only chunk rows
  int32_t n_chunk;
  uint32_t* barrier;          // grid-barrier arrival counter (monotonic, wrapping)
  uint32_t barrier_base;      // its value when this launch starts
  int32_t rows_per_block;     // set by launch_maint
  unsigned long long* moved;  // [B*Hkv] rows rewritten by staged moves (selection outcomes)
  int32_t inline_sel;         // 1: every selection is depth 0, resolved where its winner moves
};
struct MaintGrid { int blocks, rows_per_block; };
template <typename T>
cudaError_t launch_maint(const Geometry& g, const PlanDev& p, MaintItems it, StateDev<T> sd, const float* s,
                  cudaStream_t st);
// barrier arrivals one launch adds (the host advances barrier_base by it)
template <typename T>
int maint_barriers(const Geometry& g, const MaintItems& it);

void launch_positions(const Geometry& g, int32_t* pe, cudaStream_t st);

// EMA fold of every pre-chunk resident, mu <- decay*mu + s (Q4), for the paths whose
// score producer does not fold (score injection, the SIMT fp32 path); the tcgen05 pass 2
// folds in its epilogue.
void launch_ema_fold(const Geometry& g, double* mu, const float* s, cudaStream_t st);

// Homogeneous head policy: s[b][0..Hkv)[len] <- its reduction over the kv-heads
// (mode 0 max, 1 mean), written back to every kv-head.
void launch_head_homogenize(int B, int Hkv, int len, int mode, float* s, cudaStream_t st);
// homogeneous + median: s[b][g][x] = median over ALL q-heads h of heads[b][h][x], every g
void launch_head_median_all(int B, int Hq, int Hkv, int len, const float* heads, int heads_ld, float* s,
                            cudaStream_t st);

// tcgen05 attention (k_attn_tc.cu)
struct TcParams {
  int32_t B, Hq, Hkv, G, m, M, S_tot;
  int32_t Mb;                   // row stride of qbias: max_stride rounded up to 128
  float scale_log2;
  int32_t n_res_tiles;
  const int2* res_tiles;        // (start slot, valid length) of each resident key tile
  const __nv_bfloat16* q_rot;   // [B][Hq][M][D]  rotated chunk queries
  const __nv_bfloat16* k_rot;   // [B][Hkv][S_tot + M][D]  rotated keys (slot order + chunk)
  __nv_bfloat16* out;           // [B][m][Hq][D]
  float* qbias;                 // [B][Hq][Mb] lse2 - log2(w_r): log2-domain LSE of scale*log2e*S
                                //             minus the EMA row weight (+inf past m)
  const float* log2w;           // [m]  log2 of the EMA row weights
  float* s;                     // [B*Hkv][S_tot + m]
  double* mu;                   // [B*Hkv][S_tot] EMA state: pass 2 folds mu <- decay*mu + s
  double decay;                 // gamma^m
  int32_t head_reduce;          // s_g over the group: 0 max; ablations 1 mean, 2 median
  // one-pass estimator (CASCADE_OPT_ONEPASS_SCORES): pass 1 accumulates every q-head's estimated
  // mass (Alg. 3) into s_heads [B][Hq][S_tot + Mb] (zeroed per call, atomic adds)
  const float* w;               // [m] EMA row weights (1 - gamma) gamma^(m-1-r)
  float* s_heads;               // null: exact mode (pass 2)
  // homogeneous + median (P:542 ablation): pass 2 also writes every q-head's mass to
  // heads_out [B][Hq][S_tot + Mb] (null otherwise)
  float* heads_out;
};
// per-key group reduction + EMA fold of the one-pass estimates (k_attn_tc.cu)
void launch_onepass_reduce(const TcParams& p, const Geometry& g, bool fold, cudaStream_t st);
// single-token decode (k_decode.cu): one fused cluster launch per step
struct DecodeParams {
  int32_t B, Hq, Hkv, G, S_tot, alpha, N, c;
  int32_t sink_pre;
  int32_t counts[CASCADE_MAX_LEVELS], xi[CASCADE_MAX_LEVELS], base[CASCADE_MAX_LEVELS];
  int32_t n_keys;               // n_cached + 1 (the new token)
  int32_t nsplit;               // CTAs per (b, g) = cluster size
  int32_t n_tiles;              // resident key tiles (the new token is one more)
  const int4* dec_tiles;        // (start slot, length, pe of key 0, unused) per tile
  int64_t t0;                   // stream index of the new token
  float scale_log2;             // softmax scale * log2(e)
  float w0;                     // (1 - gamma): EMA weight of the single row (Alg. 3, m = 1)
  double decay;                 // gamma
  int32_t head_reduce;          // s_g over the group: 0 max; ablations 1 mean, 2 median
  int32_t homogeneous;          // head policy: 0 independent, 1 homogeneous
  int32_t update;               // fused kernel: 1 fold + insertion in-kernel; 0 s only (homogeneous)
  int32_t exact_rope;           // 1: proven-exact bf16 rounding of the rotated keys (Q17)
  const __nv_bfloat16* q;       // [B][Hq][D]   pre-RoPE
  const __nv_bfloat16* k_new;   // [B][Hkv][D]
  const __nv_bfloat16* v_new;   // [B][Hkv][D]
  __nv_bfloat16* k_raw_mut;     // state [B*Hkv][S_tot][D]
  __nv_bfloat16* v_mut;         // state
  double* mu;                   // state
  int64_t* origin;              // state
  float* s;                     // [B*Hkv][S_tot + 1] exact mass (last_scores layout)
  float* heads_out;             // homogeneous + median: every q-head's mass, row stride heads_ld
  int32_t heads_ld;
  const double2* tab;           // [npos][D/2] cos/sin(pe theta_i), fp64
  const float2* tab_hi;         // [npos/32 + 1][D] cos/sin(32 a theta_i) double-float [D/2 hi | D/2 lo]
  const float2* tab_lo;         // [32][D] cos/sin(b theta_i) double-float [D/2 hi | D/2 lo]
};
int decode_gm(int G);
size_t decode_nsplit(const DecodeParams& p);   // 0: logits of the cache do not fit in TMEM
// the fused cluster kernel (p.update: fold + insertion in-kernel, else s only)
cudaError_t launch_decode_fused(const DecodeParams& p, const PlanDev& pl, int32_t n_sel,
                                const int32_t* phase_begin_dev, int32_t n_phase, __nv_bfloat16* out,
                                const CUtensorMap& tk, const CUtensorMap& tv, cudaStream_t st);
// fold + selection + moves from s (the commit of a decode attend without inline update)
cudaError_t launch_decode_commit(const DecodeParams& p, const PlanDev& pl, int32_t n_sel,
                                 const int32_t* phase_begin_dev, int32_t n_phase, cudaStream_t st);

size_t attn_fwd_tc_smem(int d, bool est);

size_t attn_score_tc_smem(int d, int G);
void launch_attn_fwd_tc(const TcParams& p, const CUtensorMap& tq, const CUtensorMap& tk,
                        const CUtensorMap& tvs, const CUtensorMap& tvc, int d, cudaStream_t st);
void launch_attn_score_tc(const TcParams& p, const CUtensorMap& tq, const CUtensorMap& tk, int d,
                          cudaStream_t st);

}  // namespace cascade
