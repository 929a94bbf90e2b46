"""Alg. 1's layer loop over a stack of synthetic attention layers -- oracle, TEST INFRASTRUCTURE ONLY.

Alg. 1 (``alg:strided-prefill``):

    for chunk in stride(inputs, stride_size):
        for layer in model:
            KV <- cache.get()
            output, scores <- layer(chunk, KV)
            cache.update(chunk, scores)

The hot path's per-layer step (``CascadeOracle.prefill_stride``) is the ``layer(chunk, KV)``
+ ``cache.update`` pair of one attention layer.  SURVEY.md section 8(f) NEXT #4 couples the
layers the way the loop above does: layer l+1 consumes layer l's output of the SAME chunk.  The
paper's model layers are trained Llama/Qwen blocks (out of scope); the synthetic layer here is
the attention sub-layer of such a block with its projections and residual, nothing else:

    q = x W_q,  k = x W_k,  v = x W_v      (x [B, m, D] -> [B, m, H, d], pre-RoPE)
    O = cascade attention of layer l      (``CascadeOracle.prefill_stride(l, q, k, v)``)
    x <- x + O W_o                        (O [B, m, Hq d] -> [B, m, D])

Plain float64 numpy.  ``round_bf16_io`` (reading Q22) rounds every tensor the GPU
holds in bf16 between its kernels -- q, k, v, O and the residual stream x -- to bf16 at the same
points, so that per-layer checks compare the same operands; with it off the stack is exact
float64 arithmetic.
"""

from __future__ import annotations

from typing import List, Sequence

import numpy as np

from .attention import round_bf16
from .model import CascadeOracle, OracleConfig


class StackOracle:
    """A stack of ``cfg.num_layers`` synthetic attention layers, each with its own cascade."""

    def __init__(self, cfg: OracleConfig, w_q: Sequence[np.ndarray], w_k: Sequence[np.ndarray],
                 w_v: Sequence[np.ndarray], w_o: Sequence[np.ndarray], round_bf16_io: bool = False):
        L, Hq, Hk, d = cfg.num_layers, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim
        if not (len(w_q) == len(w_k) == len(w_v) == len(w_o) == L):
            raise ValueError("one weight set per layer")
        self.D = int(np.asarray(w_q[0]).shape[0])
        for l in range(L):
            if (np.shape(w_q[l]) != (self.D, Hq * d) or np.shape(w_k[l]) != (self.D, Hk * d)
                    or np.shape(w_v[l]) != (self.D, Hk * d) or np.shape(w_o[l]) != (Hq * d, self.D)):
                raise ValueError(f"layer {l}: weight shapes")
        self.cfg = cfg
        self.cas = CascadeOracle(cfg)
        f = lambda ws: [np.asarray(w, np.float64) for w in ws]
        self.w_q, self.w_k, self.w_v, self.w_o = f(w_q), f(w_k), f(w_v), f(w_o)
        self.round = round_bf16_io
        self.trace: List[dict] = []     # per layer of the last chunk: x_in, q, k, v, O, s

    def _r(self, a: np.ndarray) -> np.ndarray:
        return round_bf16(a) if self.round else a

    def project(self, layer: int, x: np.ndarray):
        """q, k, v of one layer from x [B, m, D] (the layer's input projections)."""
        cfg = self.cfg
        B, m, _ = x.shape
        q = self._r(x @ self.w_q[layer]).reshape(B, m, cfg.num_q_heads, cfg.head_dim)
        k = self._r(x @ self.w_k[layer]).reshape(B, m, cfg.num_kv_heads, cfg.head_dim)
        v = self._r(x @ self.w_v[layer]).reshape(B, m, cfg.num_kv_heads, cfg.head_dim)
        return q, k, v

    def residual(self, layer: int, x: np.ndarray, O: np.ndarray) -> np.ndarray:
        """x + O W_o (the layer's output projection and residual add)."""
        B, m, _ = x.shape
        return self._r(x + O.reshape(B, m, -1) @ self.w_o[layer])

    def prefill_stride(self, x: np.ndarray) -> np.ndarray:
        """One chunk through every layer (the inner loop of Alg. 1).  x [B, m, D] -> [B, m, D]."""
        x = self._r(np.asarray(x, np.float64))
        self.trace = []
        for l in range(self.cfg.num_layers):
            q, k, v = self.project(l, x)
            O, s = self.cas.prefill_stride(l, q, k, v)
            O = self._r(O)
            self.trace.append(dict(x=x, q=q, k=k, v=v, O=O, s=s))
            x = self.residual(l, x, O)
        return x

    def state(self, layer: int) -> dict:
        return self.cas.state(layer)


def stack_config(num_layers: int, batch: int, num_q_heads: int, num_kv_heads: int, head_dim: int,
                 sink_size: int, cache_size: int, num_cascades: int, **kw) -> OracleConfig:
    return OracleConfig(num_layers, batch, num_q_heads, num_kv_heads, head_dim, sink_size, cache_size,
                        num_cascades, **kw)
