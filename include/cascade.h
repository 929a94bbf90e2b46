/*
 * cascade.h -- C ABI of the B200 (sm_100a) Cascading KV Cache hot path.
 *
 * Method: arXiv 2406.17808, "Training-Free Exact Extension of Context Length
 * for LLMs via Cascading KV Cache".  Citations "P:n" are lines of the paper's
 * LaTeX; "Qn" are the readings listed in DESIGN.md.
 *
 * One handle holds, for every (layer l, sequence b, kv-head g), the cascade of
 * PAPER.md section 3.1: a sink buffer of alpha tokens plus N
 * sub-caches of c = |C|/N slots kept as circular buffers with an oldest-slot
 * pointer xi, the EMA score mu of every cached token
 * and its stream index ("origin").  Calls are:
 *
 *   cascade_prefill_stride  one step of Alg. 1 for one layer: the
 *                           m chunk queries attend to [sinks | cached slots |
 *                           chunk keys (causal)] (Fig. 4), the
 *                           per-key EMA mass of Alg. 3 (exact
 *                           normaliser, Q6) is reduced with max over each GQA
 *                           group, folded into mu (Q4) and the m
 *                           tokens are inserted with Alg. 2.
 *   cascade_decode          the m = 1 case (Eq. 2).
 *   cascade_state           export of the cascade state of a layer.
 *
 * Conventions shared with the oracle:
 *   flat slot of sink s          = s                       (0 <= s < alpha)
 *   flat slot of ring slot s of
 *   sub-cache i (1-indexed)      = alpha + (i-1)*c + s     (0 <= s < c)
 *   chunk row r (scores only)    = S_tot + r,  S_tot = alpha + |C|
 *   Sub-cache i accepts the token with 0-based stream index t iff
 *   t mod 2^(i-1) == 0, t counting sink insertions too (reading Q1).
 *   Selection keeps the resident on ties (strict '>').
 *   pe of a resident = its rank in [sinks; C_N oldest..newest; ...; C_1]
 *   (P:158); chunk token r gets pe = n_cached + r.  Keys are cached
 *   pre-RoPE; RoPE is rotate-half with inv_freq_i = theta^(-2i/d).
 *   The decay per chunk is g = gamma^m computed on the host in double by
 *   right-to-left binary exponentiation (result *= base when the bit is set,
 *   then base *= base); the fold is mu <- g*mu + s in IEEE double with no
 *   fused multiply-add; a new token starts at mu = s.
 *
 * Memory: the caller owns every device buffer.  The library never calls
 * cudaMalloc; it carves the caller's workspace (cascade_workspace_bytes) and
 * allocates only a small pinned host ring for schedule uploads.  All device
 * pointers must be on `device`, contiguous, 16-byte aligned (a misaligned I/O
 * pointer is INVALID_ARG, checked before anything is launched).
 *
 * Ordering: calls on one layer must be issued in order on one stream (the
 * handle keeps a host mirror of the cascade counters so no call needs a
 * device->host synchronisation).  Different layers may use different streams.
 * A handle is single-writer: do not call into one handle from two threads.
 *
 * Errors: every entry point validates on the host before launching anything;
 * a validation error (INVALID_ARG, CONFIG, SHAPE, ORDER, WORKSPACE,
 * UNSUPPORTED) leaves the device state and the host mirror untouched.  Each
 * call first clears any stale (non-sticky) CUDA error left by earlier runtime
 * calls, then checks every launch and copy it issues.  CASCADE_ERR_CUDA
 * returned before the first state-mutating kernel (the EMA fold in pass 2 or
 * the score-injection fold, maintenance, the decode update) means nothing
 * changed; once such a kernel is enqueued a CUDA error POISONS the handle:
 * the call returns CASCADE_ERR_CUDA and every later call on the handle returns
 * CASCADE_ERR_POISONED (device state and mirror may disagree; destroy the
 * handle).  Device faults surface at the next synchronisation, as CUDA does.
 */
#ifndef CASCADE_H_
#define CASCADE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CASCADE_MAX_LEVELS 16

typedef enum {
  CASCADE_OK = 0,
  CASCADE_ERR_INVALID_ARG = -1, /* null pointer, bad layer index, ...           */
  CASCADE_ERR_CONFIG = -2,      /* |C| % N != 0, gamma not in [0,1], Hq % Hkv, d */
  CASCADE_ERR_SHAPE = -3,       /* m < 1 or m > max_stride                       */
  CASCADE_ERR_ORDER = -4,       /* reserved: call out of order                   */
  CASCADE_ERR_WORKSPACE = -5,   /* workspace too small or misaligned             */
  CASCADE_ERR_CUDA = -6,        /* CUDA launch / copy error                      */
  CASCADE_ERR_UNSUPPORTED = -7, /* option not implemented in this build         */
  CASCADE_ERR_POISONED = -8     /* an earlier call failed after state-mutating   */
                                /* kernels were enqueued: destroy the handle     */
} cascade_status;

typedef enum { CASCADE_F32 = 0, CASCADE_BF16 = 1 } cascade_dtype;

typedef struct {
  int32_t num_layers;    /* L >= 1                                              */
  int32_t batch;         /* B >= 1 independent sequences                */
  int32_t num_q_heads;   /* Hq                                                  */
  int32_t num_kv_heads;  /* Hkv, Hq % Hkv == 0 (GQA); with BF16 the   */
                         /* group Hq/Hkv must be <= 8 (the tensor-core score    */
                         /* pass holds a group's partial sums in shared memory) */
                         /* else UNSUPPORTED                                    */
  int32_t head_dim;      /* d in {64, 128}                                      */
  int32_t sink_size;     /* alpha >= 0 (64 in the paper)          */
  int32_t cache_size;    /* |C| >= N, excludes the sinks (Q16)           */
  int32_t num_cascades;  /* N in [1, CASCADE_MAX_LEVELS], |C| % N == 0 (Q14)    */
  int32_t max_stride;    /* largest m a call may pass (sizes scratch)           */
  int32_t dtype;         /* cascade_dtype of q/k/v/out and the cached K/V       */
  double ema_gamma;      /* gamma in [0,1] (0.9999 in the paper)  */
  double rope_theta;     /* RoPE base > 0 (Q11)                                 */
  double softmax_scale;  /* 0 -> 1/sqrt(d) (Eq. 1)                              */
  int32_t head_policy;   /* 0 = independent heads (the paper's choice);  */
                         /* 1 = homogeneous: s reduced over all kv-heads of a   */
                         /* sequence, one decision for all (P:542 ablation;    */
                         /* needs the unsharded head set; with head_reduce 2   */
                         /* the median over all Hq <= 32 q-heads, else         */
                         /* UNSUPPORTED; cascade_update_with_scores then       */
                         /* UNSUPPORTED: kv-head s cannot give it); other      */
                         /* values CONFIG                                      */
  int32_t head_reduce;   /* 0 = max over the GQA group; the ablations   */
                         /* of P:542: 1 = mean, 2 = median (even group: mean   */
                         /* of the middle two); 1/2 need Hq/Hkv <= 32 (else    */
                         /* UNSUPPORTED); other values CONFIG                  */
  int32_t selection;     /* 1 = EMA token selection; 0 = the ablation   */
                         /* without it (reading Q3: the resident stays and the */
                         /* carried token is dropped); else CONFIG      */
  int32_t options;       /* bitmask of CASCADE_OPT_* (0: the defaults); unknown    */
                         /* bits CONFIG                                         */
} cascade_config;

/* cascade_config.options */
#define CASCADE_OPT_ONEPASS_SCORES 1     /* per-key mass by the paper's one-pass estimator  */
                                         /* (Alg. 3 normaliser l + l rho/gamma) in */
                                         /* prefill instead of the exact two-pass mass;    */
                                         /* decode stays exact.  bf16 only (else           */
                                         /* UNSUPPORTED).                                  */
#define CASCADE_OPT_EXACT_DECODE_ROPE 2  /* decode rotates cached keys with proven-exact   */
                                         /* bf16 rounding (reading Q17) at ~+45 % decode   */
                                         /* time; default: fp32 rotation, one bf16 ulp off */
                                         /* on ~2e-5 of the key elements.                  */

/* Host mirror of one layer's cascade counters (identical for all b, g). */
typedef struct {
  int64_t t;                               /* tokens offered so far            */
  int32_t sink_count;                      /* residents of the sink buffer     */
  int32_t counts[CASCADE_MAX_LEVELS];      /* residents of sub-cache i+1       */
  int32_t xi[CASCADE_MAX_LEVELS];          /* oldest slot of sub-cache i+1     */
} cascade_mirror;

typedef struct {
  cascade_mirror mirror;
  int32_t num_cascades, sub_cache_size, sink_size, slots_total; /* N, c, alpha, S_tot */
  int32_t head_dim, dtype, batch, num_kv_heads;
  int32_t n_cached;                        /* sink_count + sum(counts)          */
  /* Device pointers, layout [B][Hkv][S_tot](+[d]) for this layer:            */
  void* k_raw;        /* pre-RoPE keys, dtype                                  */
  void* v;            /* values, dtype                                         */
  double* mu;         /* EMA score, 0 for empty slots                          */
  int64_t* origin;    /* stream index, -1 for empty slots                      */
  int32_t* pe;        /* [S_tot] rank position, -1 for empty (head-independent)*/
} cascade_state_view;

typedef struct cascade_handle cascade_handle;

const char* cascade_status_string(cascade_status s);

/* Validates cfg (host only).  Returns CASCADE_OK or the error it would raise. */
cascade_status cascade_validate_config(const cascade_config* cfg);

/* Device bytes the caller must provide to cascade_init (0 if cfg is invalid). */
size_t cascade_workspace_bytes(const cascade_config* cfg);

/* Carves d_ws (ws_bytes >= cascade_workspace_bytes, 256-B aligned) and
 * initialises every cascade to empty: origin = -1, mu = 0, counters 0.  Uses
 * cudaMemsetAsync + one synchronisation (init is off the hot path).  *out is
 * a host object owned by the library; free it with cascade_destroy. */
cascade_status cascade_init(const cascade_config* cfg, void* d_ws, size_t ws_bytes,
                            int device, cascade_handle** out);

void cascade_destroy(cascade_handle* h);

/* One Alg. 1 step for one layer, all B sequences and heads.
 *   q   [B, m, Hq,  d] device, dtype   chunk queries (pre-RoPE)
 *   k   [B, m, Hkv, d] device, dtype   chunk keys (pre-RoPE; cached raw)
 *   v   [B, m, Hkv, d] device, dtype
 *   out [B, m, Hq,  d] device, dtype   attention output (written)
 *   stream: a cudaStream_t (NULL = legacy default stream).
 * Advances the layer's t by m.  Inputs are read-only and may be reused by the
 * caller as soon as the stream reaches the end of this call. */
cascade_status cascade_prefill_stride(cascade_handle* h, int32_t layer, const void* q,
                                      const void* k, const void* v, int32_t m, void* out,
                                      void* stream);

/* Same as cascade_prefill_stride but q/k/v/out are HOST buffers (pinned for
 * asynchronous copies).  The host->device and device->host copies run on
 * `stream` through a staging area inside the workspace; the call returns after
 * `out` is written (it synchronises the stream).  Calls of this variant must
 * not run concurrently on two streams of one handle. */
cascade_status cascade_prefill_stride_host(cascade_handle* h, int32_t layer, const void* q,
                                           const void* k, const void* v, int32_t m, void* out,
                                           void* stream);

/* Pipelined form of cascade_prefill_stride_host: enqueues the chunk and returns
 * without synchronising.  Host->device copies run on a library copy stream into
 * one of two staging sets (alternating per call), the step on `stream` after
 * its inputs landed, the device->host copy of `out` on a second copy stream
 * once the step is done -- so chunk c+1's inputs and chunk c-1's output move
 * over PCIe while chunk c computes.  The caller keeps q/k/v/out valid and
 * does not read `out` until cascade_host_wait returns.  One handle, one
 * stream; chunks of all layers are processed in call order. */
cascade_status cascade_prefill_stride_host_async(cascade_handle* h, int32_t layer, const void* q,
                                                 const void* k, const void* v, int32_t m, void* out,
                                                 void* stream);

/* Blocks until every copy enqueued by cascade_prefill_stride_host_async has
 * completed (all outputs are in host memory). */
cascade_status cascade_host_wait(cascade_handle* h);

/* Single-token step (Eq. 2) + update, m = 1.
 *   q [B, Hq, d], k/v [B, Hkv, d], out [B, Hq, d], device, dtype. */
cascade_status cascade_decode(cascade_handle* h, int32_t layer, const void* q, const void* k,
                              const void* v, void* out, void* stream);

/* Synchronises `stream`, writes the pe array of the layer on the device and
 * fills *out (host struct with device pointers into the workspace). */
cascade_status cascade_state(cascade_handle* h, int32_t layer, cascade_state_view* out,
                             void* stream);

/* ---- split step: attention, then (after an optional cross-device reduction of
 * the per-key mass) the cache update --------------------------------------- */

/* The two halves of one Alg. 1 step, for head policies whose per-key
 * mass must be reduced across devices: the homogeneous policy under
 * kv-head sharding needs s reduced over the kv-heads of every rank.
 *   cascade_attend   RoPE by rank, attention (out written, as cascade_prefill_stride /
 *                    cascade_decode for m = 1) and the exact per-key mass s of every
 *                    local kv-head (reduced over its GQA group; homogeneous policy: also
 *                    over the local kv-heads, so every local kv-head holds the same row).
 *                    Independent heads: the EMA fold of the residents may already be
 *                    applied (it needs no cross-device data).  No token is inserted and
 *                    the mirror does not advance.
 *   cascade_score_buffer  device pointer to the layer's s, [B][Hkv][row_len] fp32,
 *                    row_len = S_tot + m (flat slot space); the caller may reduce it in
 *                    place on `stream` (e.g. NCCL all_reduce MAX across the ranks).
 *   cascade_commit   the EMA fold (unless applied) and Alg. 2's insertion of the m
 *                    tokens from the (reduced) s; k, v must be the buffers passed to
 *                    cascade_attend, still valid; advances the mirror.
 * Between an attend and its commit every other call on that layer returns
 * CASCADE_ERR_ORDER.  cascade_prefill_stride == attend + commit. */
cascade_status cascade_attend(cascade_handle* h, int32_t layer, const void* q, const void* k,
                              const void* v, int32_t m, void* out, void* stream);
cascade_status cascade_score_buffer(cascade_handle* h, int32_t layer, float** s, int32_t* row_len);
cascade_status cascade_commit(cascade_handle* h, int32_t layer, const void* k, const void* v,
                              void* stream);

/* Checkpoint restore: overwrite one layer's cascade with `src`, a
 * state with the same geometry (num_cascades, sub_cache_size, sink_size, slots_total,
 * head_dim, dtype, batch, num_kv_heads; else CONFIG), e.g. one exported by cascade_state
 * of another handle and copied out.  src->k_raw / v [B][Hkv][S_tot][d] (dtype), mu fp64
 * and origin int64 [B][Hkv][S_tot] may be device or (pinned) host memory; they are copied
 * on `stream` (cudaMemcpyDefault).  The mirror must be reachable by Alg. 2 (sinks fill
 * first; a sub-cache that is not full holds slots [0, count) with xi = count,
 * P:160; t >= residents) else INVALID_ARG.  pe is derived, not read. */
cascade_status cascade_load_state(cascade_handle* h, int32_t layer, const cascade_state_view* src,
                                  void* stream);

/* Copies the handle's configuration into *out (host only). */
cascade_status cascade_get_config(const cascade_handle* h, cascade_config* out);

/* ---- coupled layer stack: Alg. 1's layer loop ------
 *
 * Alg. 1 runs, for every chunk, every layer of the model in order:
 * layer l+1 consumes layer l's output of the same chunk, and layer l of the next
 * chunk needs only layer l's cascade and layer l-1's output of that chunk.  A
 * cascade_stack drives the L layers of a handle as synthetic attention layers
 * with their projections and residual (the paper's model layers are trained
 * blocks, out of scope):
 *     q = x W_q, k = x W_k, v = x W_v   (plain library GEMMs, cuBLASLt, bf16 in /
 *                                         out, fp32 accumulation)
 *     out = cascade_prefill_stride(layer l, q, k, v)
 *     x  <- x + out W_o                   (cuBLASLt, residual as the C operand)
 * Each layer runs on its own stream; events order (chunk c, layer l) after (c,
 * l-1) and after layer l+1 has finished reading the residual buffer it
 * overwrites, so layer l of chunk c+1 runs while layer l+1 of chunk c does (the
 * wavefront).  bf16 handles only (else UNSUPPORTED); head_dim, heads, batch,
 * max_stride are the handle's; d_model D is free (the projections are D x H d). */
typedef struct cascade_stack cascade_stack;

typedef struct {
  const void* w_q;  /* [D, Hq*d]  row-major bf16, device                         */
  const void* w_k;  /* [D, Hkv*d]                                                */
  const void* w_v;  /* [D, Hkv*d]                                                */
  const void* w_o;  /* [Hq*d, D]                                                 */
} cascade_layer_weights;

/* Device bytes of a stack's workspace: per layer q/k/v/out scratch of max_stride
 * rows, two residual-stream buffers [B, max_stride, D] per layer boundary (L+1),
 * and a cuBLASLt workspace per layer stream.  0 if cfg is invalid or d_model < 1. */
size_t cascade_stack_workspace_bytes(const cascade_config* cfg, int32_t d_model);

/* Binds a stack to handle h (which it drives; do not call h's layers directly
 * while a stack call is in flight).  w: num_layers weight sets (device pointers
 * the caller keeps valid).  d_ws: caller-owned device workspace of at least
 * cascade_stack_workspace_bytes, 256-B aligned.  Creates L streams, events and a
 * cuBLASLt handle (host objects owned by the stack). */
cascade_status cascade_stack_init(cascade_handle* h, int32_t d_model, const cascade_layer_weights* w,
                                  void* d_ws, size_t ws_bytes, cascade_stack** out);

void cascade_stack_destroy(cascade_stack* s);

/* Strided prefill (Alg. 1) of a whole input through every layer:
 *   x [B, T, D] bf16 (device or pinned host)  -- the stream of layer-0 inputs
 *   y [B, T, D] bf16 (device or pinned host)  -- the last layer's residual stream
 * in ceil(T/m) chunks of m <= max_stride tokens (the last may be ragged).  All work
 * is enqueued before returning; `stream` waits for the last chunk's last layer
 * (which orders every layer's work of the call).  Each chunk advances every
 * layer's cascade by its length.  Errors: INVALID_ARG (null pointers), SHAPE
 * (T < 1, m < 1 or m > max_stride) before anything is enqueued; CUDA if a copy
 * or a GEMM fails, or the status of a failing cascade_prefill_stride (whose own
 * rules apply: after a state-mutating failure the handle is POISONED) -- chunks
 * before the failing one stay enqueued. */
cascade_status cascade_stack_prefill(cascade_stack* s, const void* x, int64_t T, int32_t m, void* y,
                                     void* stream);

/* Test hook: after a cascade_stack_prefill and a synchronisation, device pointers to
 * the per-layer intermediates of the LAST chunk processed (m_last rows each):
 * x_in [B,m,D] (the layer's input), q [B,m,Hq,d], k/v [B,m,Hkv,d], o [B,m,Hq,d],
 * x_out [B,m,D] (input + o W_o). */
typedef struct {
  int32_t m_last;
  void *x_in, *q, *k, *v, *o, *x_out;
} cascade_stack_view;
cascade_status cascade_stack_trace(cascade_stack* s, int32_t layer, cascade_stack_view* out);

/* ---- test hooks -------------------------------------------------------- */

/* Score injection: fold the given per-key mass and insert the m tokens, with
 * no attention.  s [B, Hkv, S_tot + m] fp32 device, flat slot space (chunk
 * row r at S_tot + r; entries of empty slots are ignored).  k/v as in
 * cascade_prefill_stride.  Used for bit-exact state parity. */
cascade_status cascade_update_with_scores(cascade_handle* h, int32_t layer, const void* k,
                                          const void* v, int32_t m, const float* s, void* stream);

/* Copies the per-key mass s of the layer's last prefill/decode into
 * out [B, Hkv, S_tot + m_last] fp32 device (flat slot space, 0 for empty slots).
 * *m_last receives that call's m. */
cascade_status cascade_last_scores(cascade_handle* h, int32_t layer, float* out, int32_t* m_last,
                                   void* stream);

/* Host-only (no device needed): advance a mirror by m insertions exactly as
 * the library does and optionally write the pe of every flat slot after the
 * advance (pe_out [S_tot], -1 for empty) and operation counts
 * (ops_out[4] = {selects, final slot writes, drops, select dependency depth}). */
cascade_status cascade_mirror_advance(const cascade_config* cfg, cascade_mirror* mirror,
                                      int32_t m, int32_t* pe_out, int64_t* ops_out);

/* Empties the cascades of one layer (mu = 0, origin = -1, counters 0) with
 * stream-ordered memsets; K/V payloads are left as they are (unreachable). */
cascade_status cascade_reset(cascade_handle* h, int32_t layer, void* stream);

/* Number of kernel launches issued by this handle since init (for the bench's
 * gpu_launches count). */
int64_t cascade_launch_count(const cascade_handle* h);

/* Kernel-class timing with CUDA events recorded on the launch stream around each
 * launch group (off by default; enabling adds event records, no synchronisation).
 * Classes: 0 rope/prep, 1 attention pass 1, 2 score pass 2, 3 maintenance (fold +
 * resolve + moves), 4 decode attention.  cascade_profile_read synchronises the
 * recorded events and returns, per class, the summed milliseconds, the number of
 * launch groups and the summed algorithmic work (flops for 1/2/4 as 4*d per visible
 * (query, key) pair; bytes for 0/3 as documented in DESIGN.md), then clears them. */
#define CASCADE_PROFILE_CLASSES 5
cascade_status cascade_profile_enable(cascade_handle* h, int32_t enable);
cascade_status cascade_profile_read(cascade_handle* h, double* ms, int64_t* count, double* work);

#ifdef __cplusplus
}
#endif

#endif /* CASCADE_H_ */
