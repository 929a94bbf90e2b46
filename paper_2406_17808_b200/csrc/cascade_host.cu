// cascade_host.cu -- the C ABI (include/cascade.h): validation, workspace carve, host
// mirror, schedule upload and the launch sequence of each call.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <type_traits>
#include <vector>

#include "internal.h"
#include "plan.h"

using namespace cascade;

namespace {

constexpr size_t kAlign = 256;
constexpr int kRing = 8;   // pinned schedule staging buffers in flight

size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }



size_t elem_size(int32_t dtype) { return dtype == CASCADE_BF16 ? 2 : 4; }

struct LayerBufs {
  // persistent state
  void* k_raw; void* v; double* mu; int64_t* origin; int32_t* pe;
  // per-call scratch (per layer so layers may run on different streams)
  float* s; float* lse; int32_t* plan; int32_t* resolved;
  float* s_heads;           // one-pass mode: per-q-head estimated mass [B][Hq][S_tot + Mb]
  float* s_allheads;        // homogeneous + median: per-q-head exact mass [B][Hq][S_tot + Mb]
  void* q_rot; void* k_rot; void* v_chunk;
  uint32_t* maint_ctl;      // [0] grid-barrier counter, then per-(b, g) 64-bit counts of rows
                            // actually rewritten (8-byte aligned)
  uint32_t maint_barrier;   // host copy of the barrier counter (wrapping)
  CUtensorMap tm_q, tm_k, tm_vs, tm_vc;   // TMA maps of q_rot, k_rot, v (state), v_chunk
  CUtensorMap tm_kraw;                    // TMA map of the pre-RoPE key state (decode)
};

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2D bf16 row-major [rows][d] map with 64 x 128 boxes and 128-byte swizzle (the UMMA K-major /
// MN-major SW128 canonical layouts).
bool make_map(CUtensorMap* map, void* base, uint64_t rows, uint32_t d) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {d, rows};
  cuuint64_t strides[1] = {(cuuint64_t)d * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct Sizes {
  size_t k_raw, v, mu, origin, pe, s, lse, plan, resolved, q_rot, k_rot, v_chunk, s_heads, s_allheads;
  size_t maint_ctl;
  size_t per_layer;
  size_t rope_tab, rope_tab_f, tab_hi, tab_lo, stage_q, stage_kv, stage_out;
  size_t total;
  int32_t plan_ints;
};

Sizes compute_sizes(const cascade_config& c) {
  Sizes z{};
  const size_t es = elem_size(c.dtype);
  const size_t B = c.batch, Hq = c.num_q_heads, Hk = c.num_kv_heads, d = c.head_dim;
  const size_t S = (size_t)c.sink_size + c.cache_size, M = c.max_stride;
  const size_t N = c.num_cascades;
  z.k_raw = align_up(B * Hk * S * d * es);
  z.v = z.k_raw;
  z.mu = align_up(B * Hk * S * 8);
  z.origin = z.mu;
  z.pe = align_up(S * 4);
  z.s = align_up(B * Hk * (S + M) * 4);
  z.lse = align_up(B * Hq * ((M + 127) / 128 * 128) * 4);
  z.s_heads = (c.options & CASCADE_OPT_ONEPASS_SCORES) ? align_up(B * Hq * (S + (M + 127) / 128 * 128) * 4) : 0;
  z.s_allheads = (c.head_policy == 1 && c.head_reduce == 2) ? align_up(B * Hq * (S + (M + 127) / 128 * 128) * 4) : 0;
  // sel (3M) + sel_order (M) + mov (2 (N+1) M) + w (M floats) + log2w (M floats)
  // + resident key tiles (2 ints each, <= S/128 + N + 2 of them)
  z.plan_ints = (int32_t)(3 * M + M + 2 * (N + 1) * M + 2 * M + 6 * (S / 128 + 2 * N + 2) + (N + 3) +
                          4 * 2 * (N + 1) * M + 48);   // + maintenance moves (4 ints each, <= 2 (N+1) M)
  z.plan = align_up((size_t)z.plan_ints * 4);
  z.resolved = align_up(B * Hk * M * 4);
  z.q_rot = align_up(B * Hq * M * d * es);
  z.k_rot = align_up(B * Hk * (S + M) * d * es);
  z.v_chunk = align_up(B * Hk * M * d * es);
  z.maint_ctl = align_up(8 + 8 * B * Hk);
  z.per_layer = z.k_raw + z.v + z.mu + z.origin + z.pe + z.s + z.lse + z.plan + z.resolved +
                z.q_rot + z.k_rot + z.v_chunk + z.maint_ctl + z.s_heads + z.s_allheads;
  z.rope_tab = align_up((S + M) * (d / 2) * sizeof(double2));
  z.rope_tab_f = align_up((S + M) * (d / 2) * sizeof(float2));
  z.tab_hi = align_up(((S + M) / 32 + 1) * d * sizeof(float2));   // [a][hi parts | lo parts]
  z.tab_lo = align_up(32 * d * sizeof(float2));
  z.stage_q = align_up(B * M * Hq * d * es);
  z.stage_kv = align_up(B * M * Hk * d * es);
  z.stage_out = z.stage_q;
  // two staging sets: the synchronous host call uses set 0, the pipelined one alternates
  z.total = z.per_layer * c.num_layers + z.rope_tab + z.rope_tab_f + z.tab_hi + z.tab_lo +
            2 * (z.stage_q + 2 * z.stage_kv + z.stage_out);
  return z;
}

}  // namespace

namespace {
// Builds the plan for the layer's next m tokens, uploads it (plus the EMA row weights) and
// advances the mirror.  Returns the device plan view and phase/depth offsets via h->plan.
struct Upload {
  PlanDev pd;
  const float* w;        // [m] EMA row weights (1 - gamma) gamma^(m-1-r)
  const float* log2w;    // [m] their log2 (-inf when w == 0)
  const int2* tiles;     // resident key tiles (start slot, valid length)
  int32_t n_tiles;
  const int32_t* phase_begin;  // plan phase offsets (N + 2 phases + end)
  const int4* dec_tiles;       // resident tiles with rank geometry (start, len, pe0, unused)
  int32_t n_dec_tiles;         // > n_tiles when full rings wrap inside a 128-slot tile
  const int4* maint_staged;    // moves that read a resident slot (MaintItems::staged)
  int32_t n_maint_staged;
  const int4* maint_chunk;     // moves that read no resident slot (MaintItems::chunk)
  int32_t n_maint_chunk;
};

// An attend (cascade_attend) whose commit is outstanding, per layer.  The host Plan is shared by
// the layers, so the pending one keeps a copy.
struct Pending {
  bool active = false;
  bool decode = false;       // fused decode attend (commit = decode_update_kernel)
  bool folded = false;       // prefill: pass 2 already folded mu (independent heads, tcgen05 path)
  int32_t m = 0;
  Geometry g{};
  Upload up{};
  cascade_mirror next{};
  Plan plan;
  DecodeParams dp{};
};
}  // namespace

struct cascade_handle {
  cascade_config cfg;
  int device;
  Sizes sz;
  int32_t alpha, N, c, S_tot;
  std::vector<LayerBufs> layers;
  std::vector<cascade_mirror> mirrors;
  std::vector<int32_t> m_last;
  std::vector<Pending> pending;   // per layer: an attend awaiting its commit
  double2* rope_tab;     // [S_tot + max_stride][d/2] (cos, sin)(pos theta_i) in fp64
  float2* rope_tab_f;    // the same rounded to fp32 (rope_prep's fast path)
  float2* tab_hi;        // [npos/32 + 1][d] (cos, sin)(32 a theta_i) double-float: [d/2 hi | d/2 lo]
  float2* tab_lo;        // [32][d] (cos, sin)(b theta_i) double-float: [d/2 hi | d/2 lo]
  void *stage_q, *stage_k, *stage_v, *stage_out;           // set 0 (aliases stage[0])
  struct Stage { void *q, *k, *v, *out; } stage[2];
  // pipelined host path (cascade_prefill_stride_host_async): copy streams and per-set events
  cudaStream_t h2d, d2h;
  cudaEvent_t ev_in[2], ev_comp[2], ev_out[2];
  bool stage_used[2];
  int host_slot;
  Planner planner;
  Plan plan;
  int32_t* pinned[kRing];
  cudaEvent_t ring_ev[kRing];
  int ring_pos;
  int64_t launches;
  // set when a CUDA error is detected after a state-mutating kernel was enqueued: the device
  // state and the host mirror may disagree, so every later call is refused (cascade.h, Errors)
  bool poisoned;
  // profiling (cascade_profile_*)
  bool profiling;
  bool nvtx;                 // CASCADE_NVTX=1: an NVTX range per launch group (ncu --nvtx, nsys)
  struct Rec { cudaEvent_t a, b; double work; };
  std::vector<Rec> recs[CASCADE_PROFILE_CLASSES];
  std::vector<cudaEvent_t> ev_pool;
  uint64_t moved_seen;      // sum over layers of the device moved-row counters at the last read
  uint64_t moved_chunk;     // chunk-row moves launched (each always rewrites its row)
  // maintenance planning scratch
  std::vector<int32_t> maint_reads;
  std::vector<int4> maint_staged, maint_chunk;
};

namespace {

cudaEvent_t pool_event(cascade_handle* h) {
  if (!h->ev_pool.empty()) { cudaEvent_t e = h->ev_pool.back(); h->ev_pool.pop_back(); return e; }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// RAII-ish scope: records a start event on construction and an end event on finish().
struct ProfScope {
  cascade_handle* h; int cls; cudaStream_t st; cudaEvent_t a = nullptr; bool pushed = false;
  ProfScope(cascade_handle* h_, int cls_, cudaStream_t st_) : h(h_), cls(cls_), st(st_) {
    static const char* const kNames[CASCADE_PROFILE_CLASSES] = {"cascade.prep", "cascade.attn_fwd",
                                                                "cascade.attn_score", "cascade.maintenance",
                                                                "cascade.decode"};
    if (h->nvtx) { nvtxRangePushA(kNames[cls]); pushed = true; }
    if (h->profiling) { a = pool_event(h); cudaEventRecord(a, st); }
  }
  ~ProfScope() {
    if (pushed) nvtxRangePop();
  }
  void finish(double work) {
    if (!a) return;
    cudaEvent_t b = pool_event(h);
    cudaEventRecord(b, st);
    h->recs[cls].push_back({a, b, work});
    a = nullptr;
  }
};

}  // namespace

extern "C" {

const char* cascade_status_string(cascade_status s) {
  switch (s) {
    case CASCADE_OK: return "ok";
    case CASCADE_ERR_INVALID_ARG: return "invalid argument";
    case CASCADE_ERR_CONFIG: return "invalid config";
    case CASCADE_ERR_SHAPE: return "bad shape (m < 1 or m > max_stride)";
    case CASCADE_ERR_ORDER: return "call out of order";
    case CASCADE_ERR_WORKSPACE: return "workspace too small or misaligned";
    case CASCADE_ERR_CUDA: return "CUDA error";
    case CASCADE_ERR_UNSUPPORTED: return "unsupported option";
    case CASCADE_ERR_POISONED: return "handle poisoned by an earlier CUDA error (destroy it)";
  }
  return "unknown status";
}

cascade_status cascade_validate_config(const cascade_config* c) {
  if (!c) return CASCADE_ERR_INVALID_ARG;
  if (c->num_layers < 1 || c->batch < 1 || c->num_q_heads < 1 || c->num_kv_heads < 1)
    return CASCADE_ERR_CONFIG;
  if (c->num_q_heads % c->num_kv_heads) return CASCADE_ERR_CONFIG;
  if (c->head_dim != 64 && c->head_dim != 128) return CASCADE_ERR_CONFIG;
  if (c->sink_size < 0 || c->num_cascades < 1 || c->num_cascades > CASCADE_MAX_LEVELS)
    return CASCADE_ERR_CONFIG;
  if (c->cache_size < c->num_cascades || c->cache_size % c->num_cascades) return CASCADE_ERR_CONFIG;
  if (!(c->ema_gamma >= 0.0 && c->ema_gamma <= 1.0)) return CASCADE_ERR_CONFIG;
  if (!(c->rope_theta > 0.0) || c->softmax_scale < 0.0) return CASCADE_ERR_CONFIG;
  if (c->max_stride < 1) return CASCADE_ERR_CONFIG;
  if (c->dtype != CASCADE_F32 && c->dtype != CASCADE_BF16) return CASCADE_ERR_CONFIG;
  if (c->selection != 0 && c->selection != 1) return CASCADE_ERR_CONFIG;
  if (c->head_reduce < 0 || c->head_reduce > 2) return CASCADE_ERR_CONFIG;
  if (c->head_reduce != 0 && c->num_q_heads / c->num_kv_heads > 32) return CASCADE_ERR_UNSUPPORTED;
  if (c->dtype == CASCADE_BF16 && c->num_q_heads / c->num_kv_heads > 8) return CASCADE_ERR_UNSUPPORTED;
  if (c->head_policy < 0 || c->head_policy > 1) return CASCADE_ERR_CONFIG;
  if (c->head_policy == 1 && c->head_reduce == 2 && c->num_q_heads > 32) return CASCADE_ERR_UNSUPPORTED;  // median of all heads
  if (c->options & ~(CASCADE_OPT_ONEPASS_SCORES | CASCADE_OPT_EXACT_DECODE_ROPE)) return CASCADE_ERR_CONFIG;
  if ((c->options & CASCADE_OPT_ONEPASS_SCORES) && c->dtype != CASCADE_BF16) return CASCADE_ERR_UNSUPPORTED;
  const long long S = (long long)c->sink_size + c->cache_size;
  if (S + c->max_stride > (1LL << 30)) return CASCADE_ERR_CONFIG;
  return CASCADE_OK;
}

size_t cascade_workspace_bytes(const cascade_config* c) {
  if (cascade_validate_config(c) != CASCADE_OK) return 0;
  return compute_sizes(*c).total;
}

cascade_status cascade_mirror_advance(const cascade_config* cfg, cascade_mirror* mirror, int32_t m,
                                      int32_t* pe_out, int64_t* ops_out) {
  cascade_status st = cascade_validate_config(cfg);
  if (st != CASCADE_OK) return st;
  if (!mirror) return CASCADE_ERR_INVALID_ARG;
  if (m < 0) return CASCADE_ERR_SHAPE;
  const int32_t N = cfg->num_cascades, c = cfg->cache_size / N;
  Planner p;
  p.configure(cfg->sink_size, N, c, cfg->selection != 0);
  Plan plan;
  p.advance(*mirror, m, ops_out ? &plan : nullptr);
  if (pe_out) mirror_positions(*mirror, cfg->sink_size, N, c, pe_out);
  if (ops_out) {
    ops_out[0] = (int64_t)plan.sel_depth.size();
    ops_out[1] = (int64_t)plan.mov.size() / 2;
    ops_out[2] = plan.drops;
    ops_out[3] = (int64_t)plan.depth_begin.size() - 1;
  }
  return CASCADE_OK;
}

void cascade_destroy(cascade_handle* h) {
  if (!h) return;
  for (auto& v : h->recs)
    for (auto& r : v) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : h->ev_pool) cudaEventDestroy(e);
  for (int i = 0; i < kRing; ++i) {
    if (h->ring_ev[i]) cudaEventDestroy(h->ring_ev[i]);
    if (h->pinned[i]) cudaFreeHost(h->pinned[i]);
  }
  if (h->h2d) { cudaStreamSynchronize(h->h2d); cudaStreamDestroy(h->h2d); }
  if (h->d2h) { cudaStreamSynchronize(h->d2h); cudaStreamDestroy(h->d2h); }
  for (int i = 0; i < 2; ++i) {
    if (h->ev_in[i]) cudaEventDestroy(h->ev_in[i]);
    if (h->ev_comp[i]) cudaEventDestroy(h->ev_comp[i]);
    if (h->ev_out[i]) cudaEventDestroy(h->ev_out[i]);
  }
  delete h;
}

cascade_status cascade_init(const cascade_config* cfg, void* d_ws, size_t ws_bytes, int device,
                            cascade_handle** out) {
  if (!cfg || !out || !d_ws) return CASCADE_ERR_INVALID_ARG;
  *out = nullptr;
  cascade_status st = cascade_validate_config(cfg);
  if (st != CASCADE_OK) return st;
  Sizes sz = compute_sizes(*cfg);
  if (ws_bytes < sz.total || (reinterpret_cast<uintptr_t>(d_ws) % kAlign)) return CASCADE_ERR_WORKSPACE;
  if (cudaSetDevice(device) != cudaSuccess) return CASCADE_ERR_CUDA;

  cascade_handle* h = new (std::nothrow) cascade_handle();
  if (!h) return CASCADE_ERR_INVALID_ARG;
  h->cfg = *cfg;
  h->device = device;
  h->sz = sz;
  h->alpha = cfg->sink_size;
  h->N = cfg->num_cascades;
  h->c = cfg->cache_size / cfg->num_cascades;
  h->S_tot = h->alpha + cfg->cache_size;
  h->planner.configure(h->alpha, h->N, h->c, h->cfg.selection != 0);
  h->launches = 0;
  h->poisoned = false;
  h->ring_pos = 0;
  h->profiling = false;
  {
    const char* e = std::getenv("CASCADE_NVTX");
    h->nvtx = e && std::atoi(e) > 0;
  }
  h->moved_seen = 0;
  h->moved_chunk = 0;
  for (int i = 0; i < kRing; ++i) { h->pinned[i] = nullptr; h->ring_ev[i] = nullptr; }

  char* p = static_cast<char*>(d_ws);
  auto take = [&](size_t n) { char* r = p; p += n; return r; };
  h->layers.resize(cfg->num_layers);
  for (auto& L : h->layers) {
    L.k_raw = take(sz.k_raw); L.v = take(sz.v);
    L.mu = reinterpret_cast<double*>(take(sz.mu));
    L.origin = reinterpret_cast<int64_t*>(take(sz.origin));
    L.pe = reinterpret_cast<int32_t*>(take(sz.pe));
    L.s = reinterpret_cast<float*>(take(sz.s));
    L.lse = reinterpret_cast<float*>(take(sz.lse));
    L.s_heads = sz.s_heads ? reinterpret_cast<float*>(take(sz.s_heads)) : nullptr;
    L.s_allheads = sz.s_allheads ? reinterpret_cast<float*>(take(sz.s_allheads)) : nullptr;
    L.plan = reinterpret_cast<int32_t*>(take(sz.plan));
    L.resolved = reinterpret_cast<int32_t*>(take(sz.resolved));
    L.q_rot = take(sz.q_rot); L.k_rot = take(sz.k_rot); L.v_chunk = take(sz.v_chunk);
    L.maint_ctl = reinterpret_cast<uint32_t*>(take(sz.maint_ctl));
    L.maint_barrier = 0;
  }
  h->rope_tab = reinterpret_cast<double2*>(take(sz.rope_tab));
  h->rope_tab_f = reinterpret_cast<float2*>(take(sz.rope_tab_f));
  h->tab_hi = reinterpret_cast<float2*>(take(sz.tab_hi));
  h->tab_lo = reinterpret_cast<float2*>(take(sz.tab_lo));
  for (int i = 0; i < 2; ++i) {
    h->stage[i].q = take(sz.stage_q); h->stage[i].k = take(sz.stage_kv);
    h->stage[i].v = take(sz.stage_kv); h->stage[i].out = take(sz.stage_out);
  }
  h->stage_q = h->stage[0].q; h->stage_k = h->stage[0].k;
  h->stage_v = h->stage[0].v; h->stage_out = h->stage[0].out;
  h->mirrors.assign(cfg->num_layers, cascade_mirror{});
  h->m_last.assign(cfg->num_layers, 0);
  h->pending.assign(cfg->num_layers, Pending{});

  bool ok = true;
  ok = ok && cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking) == cudaSuccess &&
       cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking) == cudaSuccess;
  for (int i = 0; i < 2 && ok; ++i) {
    ok = cudaEventCreateWithFlags(&h->ev_in[i], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&h->ev_comp[i], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&h->ev_out[i], cudaEventDisableTiming) == cudaSuccess;
    h->stage_used[i] = false;
  }
  h->host_slot = 0;
  for (int i = 0; i < kRing && ok; ++i) {
    ok = cudaHostAlloc(reinterpret_cast<void**>(&h->pinned[i]), (size_t)sz.plan_ints * 4,
                       cudaHostAllocDefault) == cudaSuccess &&
         cudaEventCreateWithFlags(&h->ring_ev[i], cudaEventDisableTiming) == cudaSuccess;
  }
  // Empty cascades: mu = 0, origin = -1 (all bytes 0xff), scores 0.
  for (auto& L : h->layers) {
    ok = ok && cudaMemsetAsync(L.mu, 0, sz.mu) == cudaSuccess;
    ok = ok && cudaMemsetAsync(L.origin, 0xff, sz.origin) == cudaSuccess;
    ok = ok && cudaMemsetAsync(L.k_raw, 0, sz.k_raw) == cudaSuccess;
    ok = ok && cudaMemsetAsync(L.v, 0, sz.v) == cudaSuccess;
    ok = ok && cudaMemsetAsync(L.s, 0, sz.s) == cudaSuccess;
    ok = ok && cudaMemsetAsync(L.maint_ctl, 0, sz.maint_ctl) == cudaSuccess;
    // scratch read by masked lanes of the MMAs must hold finite values (0 * NaN = NaN)
    ok = ok && cudaMemsetAsync(L.q_rot, 0, sz.q_rot) == cudaSuccess;
    ok = ok && cudaMemsetAsync(L.k_rot, 0, sz.k_rot) == cudaSuccess;
    ok = ok && cudaMemsetAsync(L.v_chunk, 0, sz.v_chunk) == cudaSuccess;
    ok = ok && cudaMemsetAsync(L.lse, 0, sz.lse) == cudaSuccess;
    if (cfg->dtype == CASCADE_BF16) {
      const uint64_t B = cfg->batch, Hq = cfg->num_q_heads, Hk = cfg->num_kv_heads, M = cfg->max_stride;
      const uint32_t d = cfg->head_dim;
      ok = ok && make_map(&L.tm_q, L.q_rot, B * Hq * M, d) &&
           make_map(&L.tm_k, L.k_rot, B * Hk * ((uint64_t)h->S_tot + M), d) &&
           make_map(&L.tm_vs, L.v, B * Hk * (uint64_t)h->S_tot, d) &&
           make_map(&L.tm_vc, L.v_chunk, B * Hk * M, d) &&
           make_map(&L.tm_kraw, L.k_raw, B * Hk * (uint64_t)h->S_tot, d);
    }
  }
  // RoPE table: (cos, sin)(pos * theta^(-2i/d)) in double (Q11); the rotation itself runs in
  // double too, so the rotated operand rounds to the same bf16 as the exact rotation (Q17)
  {
    const int half = cfg->head_dim / 2;
    const size_t npos = (size_t)h->S_tot + cfg->max_stride;
    std::vector<double2> tab(npos * half);
    for (int i = 0; i < half; ++i) {
      const double f = std::pow(cfg->rope_theta, -(2.0 * i) / cfg->head_dim);
      for (size_t pos = 0; pos < npos; ++pos) {
        const double a = (double)pos * f;
        tab[pos * half + i] = make_double2(std::cos(a), std::sin(a));
      }
    }
    ok = ok && cudaMemcpy(h->rope_tab, tab.data(), tab.size() * sizeof(double2),
                          cudaMemcpyHostToDevice) == cudaSuccess;
    std::vector<float2> tabf(tab.size());
    for (size_t e = 0; e < tab.size(); ++e) tabf[e] = make_float2((float)tab[e].x, (float)tab[e].y);
    ok = ok && cudaMemcpy(h->rope_tab_f, tabf.data(), tabf.size() * sizeof(float2),
                          cudaMemcpyHostToDevice) == cudaSuccess;
    // angle-addition factors for decode: pe = 32 a + b, cos/sin(32 a theta_i) and cos/sin(b theta_i)
    const size_t nhi = npos / 32 + 1;
    std::vector<float2> hi(nhi * 2 * half), lo(32 * 2 * half);
    auto split = [&](float2* row, int i, double a) {   // (cos, sin)(a) as fp32 hi + fp32 lo
      const double c = std::cos(a), s = std::sin(a);
      const float ch = (float)c, sh = (float)s;
      row[i] = make_float2(ch, sh);
      row[half + i] = make_float2((float)(c - (double)ch), (float)(s - (double)sh));
    };
    for (int i = 0; i < half; ++i) {
      const double f = std::pow(cfg->rope_theta, -(2.0 * i) / cfg->head_dim);
      for (size_t a = 0; a < nhi; ++a) split(&hi[a * 2 * half], i, (double)(32 * a) * f);
      for (int bb = 0; bb < 32; ++bb) split(&lo[bb * 2 * half], i, (double)bb * f);
    }
    ok = ok && cudaMemcpy(h->tab_hi, hi.data(), hi.size() * sizeof(float2), cudaMemcpyHostToDevice) == cudaSuccess;
    ok = ok && cudaMemcpy(h->tab_lo, lo.data(), lo.size() * sizeof(float2), cudaMemcpyHostToDevice) == cudaSuccess;
  }
  ok = ok && cudaDeviceSynchronize() == cudaSuccess;
  if (!ok) { cascade_destroy(h); return CASCADE_ERR_CUDA; }
  *out = h;
  return CASCADE_OK;
}

int64_t cascade_launch_count(const cascade_handle* h) { return h ? h->launches : 0; }

}  // extern "C"

namespace {

Geometry make_geometry(const cascade_handle* h, const cascade_mirror& mr, int32_t m) {
  const cascade_config& c = h->cfg;
  Geometry g{};
  g.B = c.batch; g.Hq = c.num_q_heads; g.Hkv = c.num_kv_heads; g.G = g.Hq / g.Hkv; g.d = c.head_dim;
  g.alpha = h->alpha; g.N = h->N; g.c = h->c; g.S_tot = h->S_tot;
  g.m = m; g.ldc = c.max_stride; g.t0 = mr.t; g.sink_pre = mr.sink_count;
  int32_t base = mr.sink_count, n = mr.sink_count;
  for (int i = h->N - 1; i >= 0; --i) { g.base_pre[i] = base; base += mr.counts[i]; }
  for (int i = 0; i < h->N; ++i) { g.counts_pre[i] = mr.counts[i]; g.xi_pre[i] = mr.xi[i]; n += mr.counts[i]; }
  g.n_cached = n;
  const double scale = c.softmax_scale > 0 ? c.softmax_scale : 1.0 / std::sqrt((double)c.head_dim);
  g.scale = (float)scale;
  g.scale_log2 = (float)(scale * 1.4426950408889634);
  g.decay = gamma_pow(c.ema_gamma, m);
  g.head_reduce = c.head_reduce;
  g.homogeneous = c.head_policy == 1;
  return g;
}

cascade_status upload_plan(cascade_handle* h, int32_t layer, int32_t m, cudaStream_t st,
                           Upload* up, cascade_mirror* next) {
  PlanDev* pd = &up->pd;
  const cascade_mirror pre = h->mirrors[layer];
  *next = pre;
  h->planner.advance(*next, m, &h->plan);
  const Plan& P = h->plan;
  const size_t nsel = P.sel.size(), nord = P.sel_order.size(), nmov = P.mov.size();
  // resident key tiles: valid runs (sinks, then sub-caches 1..N) cut into 128-slot tiles
  std::vector<int2> tiles;
  auto add_run = [&](int32_t beg, int32_t len) {
    for (int32_t o = 0; o < len; o += 128) tiles.push_back(make_int2(beg + o, std::min(128, len - o)));
  };
  add_run(0, pre.sink_count);
  for (int32_t i = 0; i < h->N; ++i) add_run(h->alpha + i * h->c, pre.counts[i]);
  // the same runs as 128-slot tiles with their rank geometry for decode: pe of key j = pe0 + j;
  // a tile of a full ring is split where the ring wraps past its oldest slot xi
  std::vector<int4> dt;
  for (int32_t o = 0; o < pre.sink_count; o += 128) dt.push_back(make_int4(o, std::min(128, pre.sink_count - o), o, 128));
  {
    int32_t base = pre.sink_count;
    int32_t bases[CASCADE_MAX_LEVELS];
    for (int32_t i = h->N - 1; i >= 0; --i) { bases[i] = base; base += pre.counts[i]; }
    for (int32_t i = 0; i < h->N; ++i) {
      const int32_t cnt = pre.counts[i], xi = pre.xi[i], c = h->c;
      const bool full = cnt == c;
      for (int32_t s0 = 0; s0 < cnt; s0 += 128) {
        const int32_t len = std::min(128, cnt - s0);
        const int32_t x0 = h->alpha + i * c + s0;
        if (!full) { dt.push_back(make_int4(x0, len, bases[i] + s0, 128)); continue; }
        if (s0 >= xi) { dt.push_back(make_int4(x0, len, bases[i] + s0 - xi, 128)); continue; }
        const int32_t before = std::min(len, xi - s0);         // slots s0 .. xi-1: newest part
        dt.push_back(make_int4(x0, before, bases[i] + s0 - xi + c, 128));
        if (before < len) dt.push_back(make_int4(x0 + before, len - before, bases[i], 128));
      }
    }
  }
  // maintenance moves, in phase order (C_N .. C_1, sinks): those that read a resident slot
  // (evictees, selections) and those that read only chunk rows
  const int32_t S_tot = h->S_tot;
  std::vector<int32_t>& rd = h->maint_reads;
  auto reads = [&](int32_t ref, auto&& self) -> void {    // concrete slots a reference reads
    if (ref >= 0) { if (ref < S_tot) rd.push_back(ref); return; }
    const int32_t k = -ref - 1;
    self(P.sel[3 * k + 1], self);
    self(P.sel[3 * k + 2], self);
  };
  std::vector<int4>& staged = h->maint_staged;
  std::vector<int4>& chunk_moves = h->maint_chunk;
  staged.clear();
  chunk_moves.clear();
  for (size_t e = 0; e < P.mov.size() / 2; ++e) {
    const int32_t dst = P.mov[2 * e], ref = P.mov[2 * e + 1];
    int32_t cand = 0, inc = 0;
    if (ref < 0) { cand = P.sel[3 * (-ref - 1) + 1]; inc = P.sel[3 * (-ref - 1) + 2]; }
    rd.clear();
    reads(ref, reads);
    (rd.empty() ? chunk_moves : staged).push_back(make_int4(dst, ref, cand, inc));
  }
  // layout of the upload (int32 words): sel | sel_order | mov | w [m] | log2w [m] | tiles (int2) |
  // phase_begin | dec tiles (int4) | staged moves (int4) | chunk moves (int4); every capacity is
  // checked before anything is written into the pinned buffer
  auto pad4 = [](size_t x) { return (x + 3) & ~size_t(3); };       // int2 / int4 alignment
  const size_t w_off = nsel + nord + nmov;
  const size_t tiles_off = pad4(w_off + 2 * (size_t)m);
  const size_t ph_off = tiles_off + 2 * tiles.size();
  const size_t dt_off = pad4(ph_off + P.phase_begin.size());
  const size_t mi_off = pad4(dt_off + 4 * dt.size());
  const size_t cm_off = mi_off + 4 * staged.size();
  const size_t total = cm_off + 4 * chunk_moves.size();
  if (total > (size_t)h->sz.plan_ints) return CASCADE_ERR_WORKSPACE;   // capacity formula broken
  const int slot = h->ring_pos;
  if (cudaEventSynchronize(h->ring_ev[slot]) != cudaSuccess) return CASCADE_ERR_CUDA;
  h->ring_pos = (h->ring_pos + 1) % kRing;
  int32_t* buf = h->pinned[slot];
  std::memcpy(buf, P.sel.data(), nsel * 4);
  std::memcpy(buf + nsel, P.sel_order.data(), nord * 4);
  std::memcpy(buf + nsel + nord, P.mov.data(), nmov * 4);
  float* w = reinterpret_cast<float*>(buf + w_off);
  float* lw = w + m;
  const double gam = h->cfg.ema_gamma;
  for (int32_t r = 0; r < m; ++r) {    // C_EMA = (1 - gamma) gamma^(m-1-r)  (Alg. 3)
    const double wr = (1.0 - gam) * gamma_pow(gam, m - 1 - r);
    w[r] = (float)wr;
    lw[r] = wr > 0 ? (float)std::log2(wr) : -INFINITY;
  }
  std::memcpy(buf + tiles_off, tiles.data(), tiles.size() * sizeof(int2));
  std::memcpy(buf + ph_off, P.phase_begin.data(), P.phase_begin.size() * 4);
  std::memcpy(buf + dt_off, dt.data(), dt.size() * sizeof(int4));
  std::memcpy(buf + mi_off, staged.data(), staged.size() * sizeof(int4));
  std::memcpy(buf + cm_off, chunk_moves.data(), chunk_moves.size() * sizeof(int4));
  LayerBufs& L = h->layers[layer];
  if (cudaMemcpyAsync(L.plan, buf, total * 4, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return CASCADE_ERR_CUDA;
  if (cudaEventRecord(h->ring_ev[slot], st) != cudaSuccess) return CASCADE_ERR_CUDA;
  pd->sel = L.plan;
  pd->sel_order = L.plan + nsel;
  pd->mov = L.plan + nsel + nord;
  pd->resolved = L.resolved;
  pd->sel_cap = h->cfg.max_stride;
  up->w = reinterpret_cast<const float*>(L.plan + w_off);
  up->log2w = up->w + m;
  up->tiles = reinterpret_cast<const int2*>(L.plan + tiles_off);
  up->n_tiles = (int32_t)tiles.size();
  up->phase_begin = L.plan + ph_off;
  up->dec_tiles = reinterpret_cast<const int4*>(L.plan + dt_off);
  up->n_dec_tiles = (int32_t)dt.size();
  up->maint_staged = reinterpret_cast<const int4*>(L.plan + mi_off);
  up->n_maint_staged = (int32_t)staged.size();
  up->maint_chunk = reinterpret_cast<const int4*>(L.plan + cm_off);
  up->n_maint_chunk = (int32_t)chunk_moves.size();
  return CASCADE_OK;
}

unsigned long long* maint_moved_ptr(cascade_handle* h, LayerBufs& L) {
  const size_t BG = (size_t)h->cfg.batch * h->cfg.num_kv_heads;
  (void)BG;
  return reinterpret_cast<unsigned long long*>(L.maint_ctl + 2);
}

uint64_t moved_total(cascade_handle* h) {
  uint64_t tot = 0;
  for (auto& L : h->layers) {
    const size_t BG = (size_t)h->cfg.batch * h->cfg.num_kv_heads;
    std::vector<unsigned long long> v(BG);
    cudaMemcpy(v.data(), maint_moved_ptr(h, L), 8 * BG, cudaMemcpyDeviceToHost);
    for (auto x : v) tot += x;
  }
  tot += h->moved_chunk;   // chunk-row moves always move: counted at launch
  return tot;
}

// device I/O pointers are read / written with 16-byte vectors and TMA (cascade.h: 16-B aligned)
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// row stride of the per-q-head mass buffers (s_heads, s_allheads): S_tot + max_stride rounded to 128
inline int heads_ld(const cascade_handle* h) { return h->S_tot + (h->cfg.max_stride + 127) / 128 * 128; }

// CUDA status of the launches issued since the last check (and clears it).
inline bool launches_ok() { return cudaGetLastError() == cudaSuccess; }

// A CUDA error after a state-mutating kernel was enqueued: the device state may have moved
// while the mirror did not, so the handle refuses every later call (cascade.h, Errors).
cascade_status poison(cascade_handle* h) {
  h->poisoned = true;
  return CASCADE_ERR_CUDA;
}

// Maintenance of one chunk: the EMA fold when the score producer did not fold, deep selections,
// then the cooperative move launch.  Every launch here mutates state; returns false on a launch
// error (the caller poisons the handle).
template <typename T>
bool launch_maintenance(cascade_handle* h, const Geometry& g, LayerBufs& L, const Upload& up, const Plan& P,
                        const T* k, const T* v, const float* s, bool folded, cudaStream_t st) {
  const PlanDev& pd = up.pd;
  ProfScope ps(h, 3, st);
  if (!folded) {          // the score producer did not fold mu (injection, SIMT path, homogeneous)
    launch_ema_fold(g, L.mu, s, st);
    ++h->launches;
  }
  // depth-0 selections (every selection unless m > c wraps a level inside the chunk) are
  // resolved inside the maintenance block that moves their winner; deeper ones beforehand
  const bool deep = P.depth_begin.size() > 2;
  if (deep) {
    for (size_t dpt = 0; dpt + 1 < P.depth_begin.size(); ++dpt) {
      launch_select_resolve(g, pd, P.depth_begin[dpt], P.depth_begin[dpt + 1], L.mu, s, st);
      ++h->launches;
    }
  }
  if (!launches_ok()) return false;
  MaintItems it{};
  it.inline_sel = deep ? 0 : 1;
  it.moved = maint_moved_ptr(h, L);
  it.staged = up.maint_staged;
  it.n_staged = up.n_maint_staged;
  it.chunk = up.maint_chunk;
  it.n_chunk = up.n_maint_chunk;
  it.barrier = L.maint_ctl;
  it.barrier_base = L.maint_barrier;
  StateDev<T> sd{reinterpret_cast<T*>(L.k_raw), reinterpret_cast<T*>(L.v), L.mu, L.origin, k, v};
  // the host copy of the grid-barrier counter advances only when the launch was accepted, so a
  // refused launch cannot leave the next one spinning on arrivals that never happen
  if (launch_maint<T>(g, pd, it, sd, s, st) != cudaSuccess) return false;
  L.maint_barrier += (uint32_t)maint_barriers<T>(g, it);
  h->launches += (up.n_maint_staged > 0 || up.n_maint_chunk > 0) ? 1 : 0;
  h->moved_chunk += (uint64_t)up.n_maint_chunk * g.B * g.Hkv;
  // algorithmic bytes: EMA 20 B per resident (mu r/w + s) when folded here; each row actually
  // rewritten moves K, V, mu, origin once (read + write): counted on the device (it.moved) and
  // added by cascade_profile_read
  const double bg = (double)g.B * g.Hkv;
  ps.finish(folded ? 0.0 : bg * 20.0 * g.n_cached);
  return true;
}

// The attention half of one Alg. 1 step (rows a2-a4): RoPE by rank, pass 1 (out, LSE), pass 2
// (exact per-key mass s, reduced over each GQA group; independent heads on the tcgen05 path also
// fold it into mu in pass 2's epilogue) and, homogeneous heads, the reduction of s over the
// sequence's local kv-heads.  Nothing of the cascade is inserted; *pd receives what the commit
// needs.  fold_ok = false keeps mu untouched (the split API with homogeneous heads).
template <typename T>
cascade_status attend_prefill(cascade_handle* h, int32_t layer, const T* q, const T* k, const T* v,
                              int32_t m, T* out, cudaStream_t st, Pending* pd) {
  LayerBufs& L = h->layers[layer];
  const Geometry g = make_geometry(h, h->mirrors[layer], m);
  Upload up;
  cascade_mirror next;
  cascade_status rc = upload_plan(h, layer, m, st, &up, &next);
  if (rc != CASCADE_OK) return rc;
  T* q_rot = reinterpret_cast<T*>(L.q_rot);
  T* k_rot = reinterpret_cast<T*>(L.k_rot);
  T* v_chunk = reinterpret_cast<T*>(L.v_chunk);
  const double es = sizeof(T);
  const double pairs = (double)g.B * g.Hq * ((double)m * g.n_cached + 0.5 * (double)m * (m + 1));
  const double useful = 4.0 * g.d * pairs;
  constexpr bool kTc = std::is_same<T, __nv_bfloat16>::value;
  {
    ProfScope ps(h, 0, st);
    launch_rope_prep<T>(g, q, k, v, reinterpret_cast<const T*>(L.k_raw), h->rope_tab, h->rope_tab_f, q_rot, k_rot,
                        v_chunk, st);
    ps.finish(2.0 * es * g.d * ((double)g.B * g.Hq * m + (double)g.B * g.Hkv * (g.n_cached + 2.0 * m)));
  }
  // scratch only so far (rotated operands); pass 1 writes `out` and the row LSEs
  TcParams tp{};
  if constexpr (kTc) {
    // tcgen05 path: pass 1 (O, LSE) then the key-stationary exact-mass pass 2
    tp.B = g.B; tp.Hq = g.Hq; tp.Hkv = g.Hkv; tp.G = g.G; tp.m = m; tp.M = g.ldc; tp.S_tot = g.S_tot;
    tp.Mb = (g.ldc + 127) / 128 * 128;
    tp.scale_log2 = g.scale_log2;
    tp.n_res_tiles = up.n_tiles; tp.res_tiles = up.tiles;
    tp.q_rot = q_rot; tp.k_rot = k_rot; tp.out = out; tp.qbias = L.lse; tp.log2w = up.log2w; tp.s = L.s;
    tp.mu = g.homogeneous ? nullptr : L.mu;   // pass 2 folds the EMA in its epilogue
    tp.decay = g.decay;
    tp.head_reduce = g.head_reduce;
    tp.w = up.w;
    tp.s_heads = L.s_heads;                   // non-null: the one-pass estimator (no pass 2)
    tp.heads_out = L.s_heads ? nullptr : L.s_allheads;   // homogeneous + median: every head's mass
    if (cudaMemsetAsync(L.s, 0, (size_t)g.B * g.Hkv * (g.S_tot + m) * sizeof(float), st) != cudaSuccess)
      return CASCADE_ERR_CUDA;
    if (tp.heads_out && cudaMemsetAsync(L.s_allheads, 0, h->sz.s_allheads, st) != cudaSuccess) return CASCADE_ERR_CUDA;
    if (L.s_heads && cudaMemsetAsync(L.s_heads, 0, h->sz.s_heads, st) != cudaSuccess) return CASCADE_ERR_CUDA;
    ProfScope ps(h, 1, st);
    launch_attn_fwd_tc(tp, L.tm_q, L.tm_k, L.tm_vs, L.tm_vc, g.d, st);
    ps.finish(useful);
  } else {
    ProfScope ps(h, 1, st);
    launch_attn_fwd_simt<T>(g, q_rot, k_rot, reinterpret_cast<const T*>(L.v), v_chunk, out, L.lse, st);
    ps.finish(useful);
  }
  h->launches += 2;
  if (!launches_ok()) return CASCADE_ERR_CUDA;   // nothing of the cascade state has changed yet
  // from here on a launch may mutate the cascade state (pass 2 folds mu in its epilogue)
  if constexpr (kTc) {
    if (L.s_heads) {          // one-pass estimates: group reduction (+ the fold) in one pass
      ProfScope ps(h, 2, st);
      launch_onepass_reduce(tp, g, /*fold=*/!g.homogeneous, st);
      ps.finish(0.0);
      ++h->launches;
    } else if (h->cfg.ema_gamma != 1.0) {
      ProfScope ps(h, 2, st);
      launch_attn_score_tc(tp, L.tm_q, L.tm_k, g.d, st);
      ps.finish(useful);
      ++h->launches;
    }
    // gamma = 1: every row weight (1 - gamma) gamma^k is 0, so s = 0 exactly (the memset) and
    // the fold mu <- 1 * mu + 0 leaves mu as it is; pass 2 is skipped (its FMA-pipe exp2 floors
    // at 2^-126 instead of flushing to 0, which would make the all-zero masses tiny and unequal)
  } else {
    ProfScope ps(h, 2, st);
    if (L.s_allheads && cudaMemsetAsync(L.s_allheads, 0, h->sz.s_allheads, st) != cudaSuccess)
      return CASCADE_ERR_CUDA;
    launch_attn_score_simt<T>(g, q_rot, k_rot, L.lse, up.w, L.s, L.s_allheads, heads_ld(h), st);
    ps.finish(useful);
    ++h->launches;
  }
  if (g.homogeneous) {        // one s per sequence, folded by the maintenance launch
    if (g.head_reduce == 2)     // the median of all q-heads (one-pass: of the per-head estimates)
      launch_head_median_all(g.B, g.Hq, g.Hkv, g.S_tot + m, L.s_heads ? L.s_heads : L.s_allheads, heads_ld(h),
                             L.s, st);
    else
      launch_head_homogenize(g.B, g.Hkv, g.S_tot + m, g.head_reduce, L.s, st);
    ++h->launches;
  }
  const bool folded = kTc && !g.homogeneous;
  if (!launches_ok()) return folded ? poison(h) : CASCADE_ERR_CUDA;
  pd->active = true; pd->decode = false; pd->folded = folded; pd->m = m;
  pd->g = g; pd->up = up; pd->next = next; pd->plan = h->plan;
  return CASCADE_OK;
}

// The insertion half (rows a5-a7): fold (unless pass 2 did) + Alg. 2 maintenance; commits the mirror.
template <typename T>
cascade_status commit_prefill(cascade_handle* h, int32_t layer, const T* k, const T* v, cudaStream_t st,
                              Pending& pd) {
  LayerBufs& L = h->layers[layer];
  pd.active = false;
  if (!launch_maintenance<T>(h, pd.g, L, pd.up, pd.plan, k, v, L.s, pd.folded, st) || !launches_ok())
    return poison(h);
  h->mirrors[layer] = pd.next;   // commit the mirror
  h->m_last[layer] = pd.m;
  return CASCADE_OK;
}

template <typename T>
cascade_status prefill_impl(cascade_handle* h, int32_t layer, const T* q, const T* k, const T* v,
                            int32_t m, T* out, cudaStream_t st) {
  Pending& pd = h->pending[layer];
  const cascade_status rc = attend_prefill<T>(h, layer, q, k, v, m, out, st, &pd);
  if (rc != CASCADE_OK) return rc;
  return commit_prefill<T>(h, layer, k, v, st, pd);
}

// Decode attention + mass on the fused cluster kernel.  commit_inline: the independent head
// policy lets the kernel fold and insert itself (one launch); otherwise it writes s only and
// (homogeneous heads) the local kv-heads' s are reduced, leaving the fold / selection / moves to
// commit_decode.  Returns CASCADE_ERR_UNSUPPORTED (nothing launched, mirror untouched) when the
// cache's logits do not fit in TMEM.
cascade_status attend_decode(cascade_handle* h, int32_t layer, const __nv_bfloat16* q, const __nv_bfloat16* k,
                             const __nv_bfloat16* v, __nv_bfloat16* out, cudaStream_t st, bool commit_inline,
                             Pending* pd) {
  LayerBufs& L = h->layers[layer];
  const Geometry g = make_geometry(h, h->mirrors[layer], 1);
  Upload up;
  cascade_mirror next;
  cascade_status rc = upload_plan(h, layer, 1, st, &up, &next);
  if (rc != CASCADE_OK) return rc;
  DecodeParams dp{};
  dp.B = g.B; dp.Hq = g.Hq; dp.Hkv = g.Hkv; dp.G = g.G; dp.S_tot = g.S_tot; dp.alpha = g.alpha;
  dp.N = g.N; dp.c = g.c; dp.sink_pre = g.sink_pre;
  for (int i = 0; i < g.N; ++i) { dp.counts[i] = g.counts_pre[i]; dp.xi[i] = g.xi_pre[i]; dp.base[i] = g.base_pre[i]; }
  dp.n_keys = g.n_cached + 1;
  dp.t0 = g.t0;
  dp.scale_log2 = g.scale_log2;
  dp.w0 = (float)((1.0 - h->cfg.ema_gamma) * gamma_pow(h->cfg.ema_gamma, 0));
  dp.decay = g.decay;
  dp.head_reduce = g.head_reduce;
  dp.homogeneous = g.homogeneous;
  dp.update = commit_inline && !g.homogeneous ? 1 : 0;
  dp.exact_rope = (h->cfg.options & CASCADE_OPT_EXACT_DECODE_ROPE) ? 1 : 0;
  dp.q = q; dp.k_new = k; dp.v_new = v;
  dp.k_raw_mut = static_cast<__nv_bfloat16*>(L.k_raw);
  dp.v_mut = static_cast<__nv_bfloat16*>(L.v);
  dp.mu = L.mu; dp.origin = L.origin; dp.s = L.s;
  dp.heads_out = L.s_allheads;         // homogeneous + median only (else null)
  dp.heads_ld = heads_ld(h);
  dp.tab = h->rope_tab; dp.tab_hi = h->tab_hi; dp.tab_lo = h->tab_lo;
  dp.n_tiles = up.n_dec_tiles;
  dp.dec_tiles = up.dec_tiles;
  dp.nsplit = (int32_t)decode_nsplit(dp);
  if (dp.nsplit == 0) return CASCADE_ERR_UNSUPPORTED;   // the uploaded plan is scratch
  // the kernel writes s of valid slots only: after a step of another layout (prefill rows
  // S_tot + m, injection, reset) the empty slots' entries must read 0 (cascade_last_scores)
  if (h->m_last[layer] != 1 &&
      cudaMemsetAsync(L.s, 0, (size_t)g.B * g.Hkv * (g.S_tot + 1) * sizeof(float), st) != cudaSuccess)
    return CASCADE_ERR_CUDA;
  if (L.s_allheads && cudaMemsetAsync(L.s_allheads, 0, h->sz.s_allheads, st) != cudaSuccess) return CASCADE_ERR_CUDA;
  const Plan& P = h->plan;
  {
    ProfScope ps(h, 4, st);
    const bool ok = launch_decode_fused(dp, up.pd, (int32_t)P.sel_order.size(), up.phase_begin,
                                        (int32_t)P.phase_begin.size() - 1, out, L.tm_kraw, L.tm_vs,
                                        st) == cudaSuccess;
    ++h->launches;
    if (ok && g.homogeneous) {          // one s per sequence over the local kv-heads
      if (g.head_reduce == 2)
        launch_head_median_all(g.B, g.Hq, g.Hkv, g.S_tot + 1, L.s_allheads, heads_ld(h), L.s, st);
      else
        launch_head_homogenize(g.B, g.Hkv, g.S_tot + 1, g.head_reduce, L.s, st);
      ++h->launches;
    }
    if (!ok || !launches_ok()) return dp.update ? poison(h) : CASCADE_ERR_CUDA;
    // algorithmic bytes: K, V (2 d bf16) + mu r/w + s per key
    ps.finish((double)g.B * g.Hkv * (g.n_cached + 1) * (4.0 * g.d + (dp.update ? 20.0 : 4.0)));
  }
  pd->active = true; pd->decode = true; pd->folded = false; pd->m = 1;
  pd->g = g; pd->up = up; pd->next = next; pd->plan = h->plan; pd->dp = dp;
  return CASCADE_OK;
}

cascade_status commit_decode(cascade_handle* h, int32_t layer, const __nv_bfloat16* k, const __nv_bfloat16* v,
                             cudaStream_t st, Pending& pd) {
  pd.active = false;
  if (!pd.dp.update) {                  // fold + selection + moves from s
    DecodeParams dp = pd.dp;
    dp.k_new = k; dp.v_new = v;
    ProfScope ps(h, 3, st);
    const bool ok = launch_decode_commit(dp, pd.up.pd, (int32_t)pd.plan.sel_order.size(), pd.up.phase_begin,
                                         (int32_t)pd.plan.phase_begin.size() - 1, st) == cudaSuccess;
    ++h->launches;
    if (!ok || !launches_ok()) return poison(h);
    ps.finish((double)pd.g.B * pd.g.Hkv * pd.g.n_cached * 20.0);
  }
  h->mirrors[layer] = pd.next;
  h->m_last[layer] = 1;
  return CASCADE_OK;
}

cascade_status check_call(cascade_handle* h, int32_t layer, int32_t m) {
  if (!h) return CASCADE_ERR_INVALID_ARG;
  if (h->poisoned) return CASCADE_ERR_POISONED;
  (void)cudaGetLastError();   // a stale non-sticky error of an earlier runtime call is not ours
  if (layer < 0 || layer >= h->cfg.num_layers) return CASCADE_ERR_INVALID_ARG;
  if (h->pending[layer].active) return CASCADE_ERR_ORDER;   // cascade_commit first
  if (m < 1 || m > h->cfg.max_stride) return CASCADE_ERR_SHAPE;
  return CASCADE_OK;
}

bool fused_decode_eligible(const cascade_handle* h) {
  return h->cfg.dtype == CASCADE_BF16 && h->cfg.head_dim == 128;
}

}  // namespace

extern "C" {

cascade_status cascade_prefill_stride(cascade_handle* h, int32_t layer, const void* q, const void* k,
                                      const void* v, int32_t m, void* out, void* stream) {
  cascade_status rc = check_call(h, layer, m);
  if (rc != CASCADE_OK) return rc;
  if (!q || !k || !v || !out || !aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(out)) return CASCADE_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (h->cfg.dtype == CASCADE_BF16)
    return prefill_impl<__nv_bfloat16>(h, layer, static_cast<const __nv_bfloat16*>(q),
                                       static_cast<const __nv_bfloat16*>(k),
                                       static_cast<const __nv_bfloat16*>(v), m,
                                       static_cast<__nv_bfloat16*>(out), st);
  return prefill_impl<float>(h, layer, static_cast<const float*>(q), static_cast<const float*>(k),
                             static_cast<const float*>(v), m, static_cast<float*>(out), st);
}

cascade_status cascade_prefill_stride_host(cascade_handle* h, int32_t layer, const void* q,
                                           const void* k, const void* v, int32_t m, void* out,
                                           void* stream) {
  cascade_status rc = check_call(h, layer, m);
  if (rc != CASCADE_OK) return rc;
  if (!q || !k || !v || !out) return CASCADE_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t es = elem_size(h->cfg.dtype);
  const size_t nq = (size_t)h->cfg.batch * m * h->cfg.num_q_heads * h->cfg.head_dim * es;
  const size_t nk = (size_t)h->cfg.batch * m * h->cfg.num_kv_heads * h->cfg.head_dim * es;
  // staging set 0 may still be in use by a pipelined call (its output copy is the last use)
  if (h->stage_used[0] && cudaStreamWaitEvent(st, h->ev_out[0], 0) != cudaSuccess) return CASCADE_ERR_CUDA;
  if (cudaMemcpyAsync(h->stage_q, q, nq, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(h->stage_k, k, nk, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(h->stage_v, v, nk, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return CASCADE_ERR_CUDA;
  rc = cascade_prefill_stride(h, layer, h->stage_q, h->stage_k, h->stage_v, m, h->stage_out, stream);
  if (rc != CASCADE_OK) return rc;
  if (cudaMemcpyAsync(out, h->stage_out, nq, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return CASCADE_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return CASCADE_ERR_CUDA;
  return CASCADE_OK;
}

cascade_status cascade_prefill_stride_host_async(cascade_handle* h, int32_t layer, const void* q,
                                                 const void* k, const void* v, int32_t m, void* out,
                                                 void* stream) {
  cascade_status rc = check_call(h, layer, m);
  if (rc != CASCADE_OK) return rc;
  if (!q || !k || !v || !out) return CASCADE_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t es = elem_size(h->cfg.dtype);
  const size_t nq = (size_t)h->cfg.batch * m * h->cfg.num_q_heads * h->cfg.head_dim * es;
  const size_t nk = (size_t)h->cfg.batch * m * h->cfg.num_kv_heads * h->cfg.head_dim * es;
  const int slot = h->host_slot;
  auto& S = h->stage[slot];
  // the set is free once the device->host copy of its previous chunk is done
  if (h->stage_used[slot] && cudaStreamWaitEvent(h->h2d, h->ev_out[slot], 0) != cudaSuccess) return CASCADE_ERR_CUDA;
  if (cudaMemcpyAsync(S.q, q, nq, cudaMemcpyHostToDevice, h->h2d) != cudaSuccess ||
      cudaMemcpyAsync(S.k, k, nk, cudaMemcpyHostToDevice, h->h2d) != cudaSuccess ||
      cudaMemcpyAsync(S.v, v, nk, cudaMemcpyHostToDevice, h->h2d) != cudaSuccess ||
      cudaEventRecord(h->ev_in[slot], h->h2d) != cudaSuccess ||
      cudaStreamWaitEvent(st, h->ev_in[slot], 0) != cudaSuccess)
    return CASCADE_ERR_CUDA;
  rc = cascade_prefill_stride(h, layer, S.q, S.k, S.v, m, S.out, stream);
  if (rc != CASCADE_OK) return rc;
  if (cudaEventRecord(h->ev_comp[slot], st) != cudaSuccess ||
      cudaStreamWaitEvent(h->d2h, h->ev_comp[slot], 0) != cudaSuccess ||
      cudaMemcpyAsync(out, S.out, nq, cudaMemcpyDeviceToHost, h->d2h) != cudaSuccess ||
      cudaEventRecord(h->ev_out[slot], h->d2h) != cudaSuccess)
    return CASCADE_ERR_CUDA;
  h->stage_used[slot] = true;
  h->host_slot ^= 1;
  return CASCADE_OK;
}

cascade_status cascade_host_wait(cascade_handle* h) {
  if (!h) return CASCADE_ERR_INVALID_ARG;
  if (cudaStreamSynchronize(h->h2d) != cudaSuccess || cudaStreamSynchronize(h->d2h) != cudaSuccess)
    return CASCADE_ERR_CUDA;
  return CASCADE_OK;
}

cascade_status cascade_decode(cascade_handle* h, int32_t layer, const void* q, const void* k,
                              const void* v, void* out, void* stream) {
  // q [B,Hq,d] is [B,1,Hq,d]: the m = 1 case of the strided step (Eq. 2).
  // bf16 with d = 128 (the Llama shapes, any GQA group <= 8) runs the fused cluster decode kernel
  // (one launch); the fp32 toy, d = 64 and caches whose logits do not fit in TMEM run the m = 1
  // case of the strided kernels.
  if (h == nullptr || !fused_decode_eligible(h)) return cascade_prefill_stride(h, layer, q, k, v, 1, out, stream);
  cascade_status rc = check_call(h, layer, 1);
  if (rc != CASCADE_OK) return rc;
  if (!q || !k || !v || !out || !aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(out)) return CASCADE_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const auto* kb = static_cast<const __nv_bfloat16*>(k);
  const auto* vb = static_cast<const __nv_bfloat16*>(v);
  Pending& pd = h->pending[layer];
  rc = attend_decode(h, layer, static_cast<const __nv_bfloat16*>(q), kb, vb, static_cast<__nv_bfloat16*>(out),
                     st, /*commit_inline=*/true, &pd);
  if (rc == CASCADE_ERR_UNSUPPORTED) return cascade_prefill_stride(h, layer, q, k, v, 1, out, stream);
  if (rc != CASCADE_OK) return rc;
  return commit_decode(h, layer, kb, vb, st, pd);
}

cascade_status cascade_attend(cascade_handle* h, int32_t layer, const void* q, const void* k, const void* v,
                              int32_t m, void* out, void* stream) {
  cascade_status rc = check_call(h, layer, m);
  if (rc != CASCADE_OK) return rc;
  if (!q || !k || !v || !out || !aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(out)) return CASCADE_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Pending& pd = h->pending[layer];
  if (m == 1 && fused_decode_eligible(h)) {
    rc = attend_decode(h, layer, static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k),
                       static_cast<const __nv_bfloat16*>(v), static_cast<__nv_bfloat16*>(out), st,
                       /*commit_inline=*/false, &pd);
    if (rc != CASCADE_ERR_UNSUPPORTED) return rc;
  }
  if (h->cfg.dtype == CASCADE_BF16)
    return attend_prefill<__nv_bfloat16>(h, layer, static_cast<const __nv_bfloat16*>(q),
                                         static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(v),
                                         m, static_cast<__nv_bfloat16*>(out), st, &pd);
  return attend_prefill<float>(h, layer, static_cast<const float*>(q), static_cast<const float*>(k),
                               static_cast<const float*>(v), m, static_cast<float*>(out), st, &pd);
}

cascade_status cascade_score_buffer(cascade_handle* h, int32_t layer, float** s, int32_t* row_len) {
  if (!h || !s || !row_len || layer < 0 || layer >= h->cfg.num_layers) return CASCADE_ERR_INVALID_ARG;
  const Pending& pd = h->pending[layer];
  if (!pd.active) return CASCADE_ERR_ORDER;
  *s = h->layers[layer].s;
  *row_len = h->S_tot + pd.m;
  return CASCADE_OK;
}

cascade_status cascade_commit(cascade_handle* h, int32_t layer, const void* k, const void* v, void* stream) {
  if (!h || !k || !v || !aligned16(k) || !aligned16(v) || layer < 0 || layer >= h->cfg.num_layers) return CASCADE_ERR_INVALID_ARG;
  if (h->poisoned) return CASCADE_ERR_POISONED;
  (void)cudaGetLastError();
  Pending& pd = h->pending[layer];
  if (!pd.active) return CASCADE_ERR_ORDER;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (pd.decode)
    return commit_decode(h, layer, static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(v), st, pd);
  if (h->cfg.dtype == CASCADE_BF16)
    return commit_prefill<__nv_bfloat16>(h, layer, static_cast<const __nv_bfloat16*>(k),
                                         static_cast<const __nv_bfloat16*>(v), st, pd);
  return commit_prefill<float>(h, layer, static_cast<const float*>(k), static_cast<const float*>(v), st, pd);
}

cascade_status cascade_update_with_scores(cascade_handle* h, int32_t layer, const void* k,
                                          const void* v, int32_t m, const float* s, void* stream) {
  cascade_status rc = check_call(h, layer, m);
  if (rc != CASCADE_OK) return rc;
  if (!k || !v || !s || !aligned16(k) || !aligned16(v) || !aligned16(s)) return CASCADE_ERR_INVALID_ARG;
  // the median of all q-heads (homogeneous + median) is not a function of per-kv-head s
  if (h->cfg.head_policy == 1 && h->cfg.head_reduce == 2) return CASCADE_ERR_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  LayerBufs& L = h->layers[layer];
  const Geometry g = make_geometry(h, h->mirrors[layer], m);
  Upload up;
  cascade_mirror next;
  rc = upload_plan(h, layer, m, st, &up, &next);
  if (rc != CASCADE_OK) return rc;
  const PlanDev& pd = up.pd;
  if (g.homogeneous) {        // the injected kv-head scores reduced per sequence
    const size_t n = (size_t)g.B * g.Hkv * (g.S_tot + m);
    if (cudaMemcpyAsync(L.s, s, n * sizeof(float), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return CASCADE_ERR_CUDA;
    launch_head_homogenize(g.B, g.Hkv, g.S_tot + m, g.head_reduce, L.s, st);
    ++h->launches;
    if (!launches_ok()) return CASCADE_ERR_CUDA;   // scratch only so far
    s = L.s;
  }
  const bool ok = h->cfg.dtype == CASCADE_BF16
                      ? launch_maintenance<__nv_bfloat16>(h, g, L, up, h->plan, static_cast<const __nv_bfloat16*>(k),
                                                          static_cast<const __nv_bfloat16*>(v), s, false, st)
                      : launch_maintenance<float>(h, g, L, up, h->plan, static_cast<const float*>(k),
                                                  static_cast<const float*>(v), s, false, st);
  if (!ok || !launches_ok()) return poison(h);
  h->mirrors[layer] = next;
  h->m_last[layer] = 0;
  return CASCADE_OK;
}

cascade_status cascade_last_scores(cascade_handle* h, int32_t layer, float* out, int32_t* m_last,
                                   void* stream) {
  if (!h || !out || layer < 0 || layer >= h->cfg.num_layers) return CASCADE_ERR_INVALID_ARG;
  const int32_t m = h->m_last[layer];
  if (m_last) *m_last = m;
  if (m == 0) return CASCADE_ERR_ORDER;
  const size_t n = (size_t)h->cfg.batch * h->cfg.num_kv_heads * (h->S_tot + m);
  if (cudaMemcpyAsync(out, h->layers[layer].s, n * 4, cudaMemcpyDeviceToDevice,
                      static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return CASCADE_ERR_CUDA;
  return CASCADE_OK;
}

cascade_status cascade_reset(cascade_handle* h, int32_t layer, void* stream) {
  if (!h || layer < 0 || layer >= h->cfg.num_layers) return CASCADE_ERR_INVALID_ARG;
  if (h->poisoned) return CASCADE_ERR_POISONED;
  if (h->pending[layer].active) return CASCADE_ERR_ORDER;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  LayerBufs& L = h->layers[layer];
  if (cudaMemsetAsync(L.mu, 0, h->sz.mu, st) != cudaSuccess ||
      cudaMemsetAsync(L.origin, 0xff, h->sz.origin, st) != cudaSuccess ||
      cudaMemsetAsync(L.s, 0, h->sz.s, st) != cudaSuccess ||         // decode writes valid slots only
      cudaMemsetAsync(L.maint_ctl, 0, 4, st) != cudaSuccess)   // the barrier; the moved-row counts
                                                               // keep running
    return CASCADE_ERR_CUDA;
  L.maint_barrier = 0;
  h->mirrors[layer] = cascade_mirror{};
  h->m_last[layer] = 0;
  return CASCADE_OK;
}

cascade_status cascade_profile_enable(cascade_handle* h, int32_t enable) {
  if (!h) return CASCADE_ERR_INVALID_ARG;
  h->profiling = enable != 0;
  if (cudaDeviceSynchronize() != cudaSuccess) return CASCADE_ERR_CUDA;
  h->moved_seen = moved_total(h);
  return CASCADE_OK;
}

cascade_status cascade_profile_read(cascade_handle* h, double* ms, int64_t* count, double* work) {
  if (!h || !ms || !count || !work) return CASCADE_ERR_INVALID_ARG;
  for (int c = 0; c < CASCADE_PROFILE_CLASSES; ++c) {
    ms[c] = 0; count[c] = 0; work[c] = 0;
    for (auto& r : h->recs[c]) {
      float t = 0.f;
      if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess)
        return CASCADE_ERR_CUDA;
      ms[c] += t; count[c] += 1; work[c] += r.work;
      h->ev_pool.push_back(r.a); h->ev_pool.push_back(r.b);
    }
    h->recs[c].clear();
  }
  // maintenance rows actually rewritten since the last read: K, V (d elements each), mu and
  // origin (8 B each), read once and written once
  const uint64_t now = moved_total(h);
  const double row = 2.0 * (2.0 * h->cfg.head_dim * (double)elem_size(h->cfg.dtype) + 16.0);
  work[3] += row * (double)(now - h->moved_seen);
  h->moved_seen = now;
  return CASCADE_OK;
}

cascade_status cascade_load_state(cascade_handle* h, int32_t layer, const cascade_state_view* src, void* stream) {
  if (!h || !src || layer < 0 || layer >= h->cfg.num_layers) return CASCADE_ERR_INVALID_ARG;
  if (h->poisoned) return CASCADE_ERR_POISONED;
  if (h->pending[layer].active) return CASCADE_ERR_ORDER;
  (void)cudaGetLastError();
  const cascade_config& c = h->cfg;
  if (src->num_cascades != h->N || src->sub_cache_size != h->c || src->sink_size != h->alpha ||
      src->slots_total != h->S_tot || src->head_dim != c.head_dim || src->dtype != c.dtype ||
      src->batch != c.batch || src->num_kv_heads != c.num_kv_heads)
    return CASCADE_ERR_CONFIG;
  if (!src->k_raw || !src->v || !src->mu || !src->origin) return CASCADE_ERR_INVALID_ARG;
  // the mirror must be one Alg. 2 can reach: sinks fill first, a sub-cache that is not
  // full holds slots [0, count) with xi = count, the counters fit the stream so far
  const cascade_mirror& mr = src->mirror;
  int64_t n = mr.sink_count;
  if (mr.sink_count < 0 || mr.sink_count > h->alpha) return CASCADE_ERR_INVALID_ARG;
  for (int i = 0; i < CASCADE_MAX_LEVELS; ++i) {
    const int32_t cnt = mr.counts[i], xi = mr.xi[i];
    if (i >= h->N) { if (cnt || xi) return CASCADE_ERR_INVALID_ARG; continue; }
    if (cnt < 0 || cnt > h->c || xi < 0 || xi >= h->c) return CASCADE_ERR_INVALID_ARG;
    if (cnt < h->c && xi != cnt % h->c) return CASCADE_ERR_INVALID_ARG;
    if (cnt > 0 && mr.sink_count < h->alpha) return CASCADE_ERR_INVALID_ARG;
    n += cnt;
  }
  if (mr.t < n) return CASCADE_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  LayerBufs& L = h->layers[layer];
  const size_t rows = (size_t)c.batch * c.num_kv_heads * h->S_tot;
  const size_t row_bytes = (size_t)c.head_dim * elem_size(c.dtype);
  if (cudaMemcpyAsync(L.k_raw, src->k_raw, rows * row_bytes, cudaMemcpyDefault, st) != cudaSuccess ||
      cudaMemcpyAsync(L.v, src->v, rows * row_bytes, cudaMemcpyDefault, st) != cudaSuccess ||
      cudaMemcpyAsync(L.mu, src->mu, rows * 8, cudaMemcpyDefault, st) != cudaSuccess ||
      cudaMemcpyAsync(L.origin, src->origin, rows * 8, cudaMemcpyDefault, st) != cudaSuccess ||
      cudaMemsetAsync(L.s, 0, h->sz.s, st) != cudaSuccess)
    return poison(h);   // a partial copy leaves the layer neither old nor new
  h->mirrors[layer] = mr;
  h->m_last[layer] = 0;
  return CASCADE_OK;
}

cascade_status cascade_get_config(const cascade_handle* h, cascade_config* out) {
  if (!h || !out) return CASCADE_ERR_INVALID_ARG;
  *out = h->cfg;
  return CASCADE_OK;
}

cascade_status cascade_state(cascade_handle* h, int32_t layer, cascade_state_view* out, void* stream) {
  if (!h || !out || layer < 0 || layer >= h->cfg.num_layers) return CASCADE_ERR_INVALID_ARG;
  if (h->poisoned) return CASCADE_ERR_POISONED;
  if (h->pending[layer].active) return CASCADE_ERR_ORDER;
  (void)cudaGetLastError();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  LayerBufs& L = h->layers[layer];
  const cascade_mirror& mr = h->mirrors[layer];
  const Geometry g = make_geometry(h, mr, 1);
  launch_positions(g, L.pe, st);
  ++h->launches;
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess)
    return CASCADE_ERR_CUDA;
  std::memset(out, 0, sizeof(*out));
  out->mirror = mr;
  out->num_cascades = h->N; out->sub_cache_size = h->c; out->sink_size = h->alpha;
  out->slots_total = h->S_tot; out->head_dim = h->cfg.head_dim; out->dtype = h->cfg.dtype;
  out->batch = h->cfg.batch; out->num_kv_heads = h->cfg.num_kv_heads;
  out->n_cached = g.n_cached;
  out->k_raw = L.k_raw; out->v = L.v; out->mu = L.mu; out->origin = L.origin; out->pe = L.pe;
  return CASCADE_OK;
}

}  // extern "C"
