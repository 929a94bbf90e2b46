// stack.cu -- coupled layer stack: Alg. 1's layer loop as a wavefront over
// per-layer streams.  Host code only: the projections are plain
// library GEMMs (cuBLASLt, bf16 in/out, fp32 accumulation); every layer's attention and cache
// update is cascade_prefill_stride on the layer's stream.
//
// Dependencies per (chunk c, layer l), all on the device (events, no host waits):
//   * input   X[l][c % 2]  -- written by (c, l-1) (l = 0: gathered from the caller's x on
//                            layer 0's stream, right before);
//   * output  X[l+1][c % 2] -- last read by (c-2, l+1): its QKV projections and its residual;
//   * cascade of layer l   -- (c-1, l), the previous work on the same stream.
// So (c+1, l) runs next to (c, l+1): layers of consecutive chunks overlap along the diagonal.
// One event per (layer, ring slot) records "(c, l) finished": it is both "X[l+1][slot] holds
// chunk c" for layer l+1 and "X[l][slot] is free" for layer l-1 two chunks later.
#include <cublasLt.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <tuple>
#include <vector>

#include "../../include/cascade.h"

namespace {

constexpr size_t kAlign = 256;
constexpr size_t kLtWorkspace = 4u << 20;   // per layer stream
constexpr int kSlots = 2;                    // residual-stream ring depth (chunks in flight)

size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct StackSizes {
  size_t x, q, kv, o, lt, per_layer, total;
};

StackSizes stack_sizes(const cascade_config& c, int32_t D) {
  StackSizes z{};
  const size_t rows = (size_t)c.batch * c.max_stride, es = 2;
  z.x = align_up(rows * D * es);
  z.q = align_up(rows * c.num_q_heads * c.head_dim * es);
  z.kv = align_up(rows * c.num_kv_heads * c.head_dim * es);
  z.o = z.q;
  z.lt = align_up(kLtWorkspace);
  z.per_layer = z.q + 2 * z.kv + z.o + z.lt;
  z.total = (size_t)(c.num_layers + 1) * kSlots * z.x + (size_t)c.num_layers * z.per_layer;
  return z;
}

}  // namespace

struct cascade_stack {
  cascade_handle* h;
  cascade_config cfg;
  int32_t D;
  std::vector<cascade_layer_weights> w;
  cublasLtHandle_t lt;
  std::vector<cudaStream_t> st;               // one per layer
  std::vector<cudaEvent_t> done;              // [L][kSlots]: (c, l) finished
  cudaEvent_t ev_start;
  std::vector<uint8_t*> X;                    // [(L+1)][kSlots] residual-stream buffers
  std::vector<uint8_t*> q, k, v, o, ltws;     // per layer
  int64_t chunk_ctr;                          // chunks processed over the stack's life
  int32_t m_last;
  // cuBLASLt algorithm per (rows, cin, cout, residual)
  std::map<std::tuple<int, int, int, int>, cublasLtMatmulAlgo_t> algos;
};

namespace {

// Y[R x Cout] = X[R x Cin] @ W[Cin x Cout] (+ Res[R x Cout]), all row-major bf16.  In cuBLASLt's
// column-major terms: Y^T = W^T X^T with W^T (Cout x Cin, ld Cout), X^T (Cin x R, ld Cin).
cascade_status gemm(cascade_stack* s, int layer, const void* Xp, const void* Wp, const void* Res, void* Y,
                    int R, int Cin, int Cout, cudaStream_t stream) {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  cascade_status rc = CASCADE_ERR_CUDA;
  const float alpha = 1.f, beta = Res ? 1.f : 0.f;
  do {
    if (cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F) != CUBLAS_STATUS_SUCCESS) break;
    if (cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, Cout, Cin, Cout) != CUBLAS_STATUS_SUCCESS) break;
    if (cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, Cin, R, Cin) != CUBLAS_STATUS_SUCCESS) break;
    if (cublasLtMatrixLayoutCreate(&lc, CUDA_R_16BF, Cout, R, Cout) != CUBLAS_STATUS_SUCCESS) break;
    const auto key = std::make_tuple(R, Cin, Cout, Res ? 1 : 0);
    auto it = s->algos.find(key);
    if (it == s->algos.end()) {
      cublasLtMatmulPreference_t pref = nullptr;
      if (cublasLtMatmulPreferenceCreate(&pref) != CUBLAS_STATUS_SUCCESS) break;
      size_t ws = kLtWorkspace;
      cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws, sizeof(ws));
      cublasLtMatmulHeuristicResult_t res{};
      int found = 0;
      const cublasStatus_t hs = cublasLtMatmulAlgoGetHeuristic(s->lt, op, la, lb, lc, lc, pref, 1, &res, &found);
      cublasLtMatmulPreferenceDestroy(pref);
      if (hs != CUBLAS_STATUS_SUCCESS || found < 1) break;
      it = s->algos.emplace(key, res.algo).first;
    }
    if (cublasLtMatmul(s->lt, op, &alpha, Wp, la, Xp, lb, &beta, Res ? Res : Y, lc, Y, lc, &it->second,
                       s->ltws[layer], kLtWorkspace, stream) != CUBLAS_STATUS_SUCCESS)
      break;
    rc = CASCADE_OK;
  } while (false);
  if (lc) cublasLtMatrixLayoutDestroy(lc);
  if (lb) cublasLtMatrixLayoutDestroy(lb);
  if (la) cublasLtMatrixLayoutDestroy(la);
  if (op) cublasLtMatmulDescDestroy(op);
  return rc;
}

}  // namespace

extern "C" {

size_t cascade_stack_workspace_bytes(const cascade_config* cfg, int32_t d_model) {
  if (!cfg || d_model < 1 || cascade_validate_config(cfg) != CASCADE_OK) return 0;
  return stack_sizes(*cfg, d_model).total;
}

void cascade_stack_destroy(cascade_stack* s) {
  if (!s) return;
  for (auto e : s->done)
    if (e) cudaEventDestroy(e);
  if (s->ev_start) cudaEventDestroy(s->ev_start);
  for (auto x : s->st)
    if (x) cudaStreamDestroy(x);
  if (s->lt) cublasLtDestroy(s->lt);
  delete s;
}

cascade_status cascade_stack_init(cascade_handle* h, int32_t d_model, const cascade_layer_weights* w,
                                  void* d_ws, size_t ws_bytes, cascade_stack** out) {
  if (!h || !w || !out || d_model < 1) return CASCADE_ERR_INVALID_ARG;
  *out = nullptr;
  cascade_config cfg;
  if (cascade_get_config(h, &cfg) != CASCADE_OK) return CASCADE_ERR_INVALID_ARG;
  if (cfg.dtype != CASCADE_BF16) return CASCADE_ERR_UNSUPPORTED;
  const StackSizes z = stack_sizes(cfg, d_model);
  if (!d_ws || ws_bytes < z.total || (reinterpret_cast<uintptr_t>(d_ws) % kAlign)) return CASCADE_ERR_WORKSPACE;
  const int L = cfg.num_layers;
  for (int l = 0; l < L; ++l)
    if (!w[l].w_q || !w[l].w_k || !w[l].w_v || !w[l].w_o) return CASCADE_ERR_INVALID_ARG;
  cascade_stack* s = new cascade_stack();
  s->h = h; s->cfg = cfg; s->D = d_model;
  s->w.assign(w, w + L);
  s->lt = nullptr; s->ev_start = nullptr; s->chunk_ctr = 0; s->m_last = 0;
  bool ok = cublasLtCreate(&s->lt) == CUBLAS_STATUS_SUCCESS;
  s->st.assign(L, nullptr);
  s->done.assign((size_t)L * kSlots, nullptr);
  for (int l = 0; ok && l < L; ++l) ok = cudaStreamCreateWithFlags(&s->st[l], cudaStreamNonBlocking) == cudaSuccess;
  for (auto& e : s->done)
    if (ok) ok = cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
  if (ok) ok = cudaEventCreateWithFlags(&s->ev_start, cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    cascade_stack_destroy(s);
    return CASCADE_ERR_CUDA;
  }
  uint8_t* p = static_cast<uint8_t*>(d_ws);
  auto take = [&](size_t n) { uint8_t* r = p; p += n; return r; };
  for (int i = 0; i < (L + 1) * kSlots; ++i) s->X.push_back(take(z.x));
  for (int l = 0; l < L; ++l) {
    s->q.push_back(take(z.q)); s->k.push_back(take(z.kv)); s->v.push_back(take(z.kv));
    s->o.push_back(take(z.o)); s->ltws.push_back(take(z.lt));
  }
  *out = s;
  return CASCADE_OK;
}

cascade_status cascade_stack_prefill(cascade_stack* s, const void* x, int64_t T, int32_t m, void* y, void* stream) {
  if (!s || !x || !y) return CASCADE_ERR_INVALID_ARG;
  if (T < 1 || m < 1 || m > s->cfg.max_stride) return CASCADE_ERR_SHAPE;
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  const cascade_config& c = s->cfg;
  const int L = c.num_layers, B = c.batch, D = s->D;
  const int Hq = c.num_q_heads, Hk = c.num_kv_heads, d = c.head_dim;
  const size_t es = 2, row = (size_t)D * es;
  cudaGetLastError();
  if (cudaEventRecord(s->ev_start, cs) != cudaSuccess) return CASCADE_ERR_CUDA;
  for (int l = 0; l < L; ++l)       // the caller's prior work (x written, y free) comes first
    if (cudaStreamWaitEvent(s->st[l], s->ev_start, 0) != cudaSuccess) return CASCADE_ERR_CUDA;
  const int64_t nchunks = (T + m - 1) / m;
  int slot = 0;
  for (int64_t ci = 0; ci < nchunks; ++ci) {
    const int64_t t0 = ci * m;
    const int mc = (int)std::min<int64_t>(m, T - t0);
    const int64_t cg = s->chunk_ctr++;
    slot = (int)(cg % kSlots);
    const int R = B * mc;
    for (int l = 0; l < L; ++l) {
      cudaStream_t st = s->st[l];
      uint8_t* xin = s->X[(size_t)l * kSlots + slot];
      uint8_t* xout = s->X[(size_t)(l + 1) * kSlots + slot];
      if (l == 0) {   // gather the chunk's rows of every sequence: [B, mc, D] from [B, T, D]
        if (cudaMemcpy2DAsync(xin, mc * row, static_cast<const uint8_t*>(x) + t0 * row, (size_t)T * row, mc * row, B,
                              cudaMemcpyDefault, st) != cudaSuccess)
          return CASCADE_ERR_CUDA;
      } else if (cudaStreamWaitEvent(st, s->done[(size_t)(l - 1) * kSlots + slot], 0) != cudaSuccess) {
        return CASCADE_ERR_CUDA;
      }
      // X[l+1][slot] was last read by (c-2, l+1)
      if (cg >= kSlots && l + 1 < L &&
          cudaStreamWaitEvent(st, s->done[(size_t)(l + 1) * kSlots + slot], 0) != cudaSuccess)
        return CASCADE_ERR_CUDA;
      const cascade_layer_weights& w = s->w[l];
      cascade_status rc;
      if ((rc = gemm(s, l, xin, w.w_q, nullptr, s->q[l], R, D, Hq * d, st)) != CASCADE_OK) return rc;
      if ((rc = gemm(s, l, xin, w.w_k, nullptr, s->k[l], R, D, Hk * d, st)) != CASCADE_OK) return rc;
      if ((rc = gemm(s, l, xin, w.w_v, nullptr, s->v[l], R, D, Hk * d, st)) != CASCADE_OK) return rc;
      if ((rc = cascade_prefill_stride(s->h, l, s->q[l], s->k[l], s->v[l], mc, s->o[l], st)) != CASCADE_OK) return rc;
      if ((rc = gemm(s, l, s->o[l], w.w_o, xin, xout, R, Hq * d, D, st)) != CASCADE_OK) return rc;
      if (l == L - 1 &&   // scatter the chunk into y [B, T, D]
          cudaMemcpy2DAsync(static_cast<uint8_t*>(y) + t0 * row, (size_t)T * row, xout, mc * row, mc * row, B,
                            cudaMemcpyDefault, st) != cudaSuccess)
        return CASCADE_ERR_CUDA;
      if (cudaEventRecord(s->done[(size_t)l * kSlots + slot], st) != cudaSuccess) return CASCADE_ERR_CUDA;
    }
    s->m_last = mc;
  }
  if (cudaStreamWaitEvent(cs, s->done[(size_t)(L - 1) * kSlots + slot], 0) != cudaSuccess) return CASCADE_ERR_CUDA;
  return cudaGetLastError() == cudaSuccess ? CASCADE_OK : CASCADE_ERR_CUDA;
}

cascade_status cascade_stack_trace(cascade_stack* s, int32_t layer, cascade_stack_view* out) {
  if (!s || !out || layer < 0 || layer >= s->cfg.num_layers) return CASCADE_ERR_INVALID_ARG;
  if (s->chunk_ctr == 0) return CASCADE_ERR_ORDER;
  const int slot = (int)((s->chunk_ctr - 1) % kSlots);
  out->m_last = s->m_last;
  out->x_in = s->X[(size_t)layer * kSlots + slot];
  out->x_out = s->X[(size_t)(layer + 1) * kSlots + slot];
  out->q = s->q[layer]; out->k = s->k[layer]; out->v = s->v[layer]; out->o = s->o[layer];
  return CASCADE_OK;
}

}  // extern "C"
