"""Seeded synthetic Q/K/V generator shared by the tests, the bench and smoke().

Holds none of the method's arithmetic: it only draws random tensors with the
structure DESIGN.md "Input recipe" describes (Llama-like head shapes, a salience
direction that makes EMA scores well separated, an optional passkey block).

Recipe (per sequence b, stream position j, kv-head g, q-head h):
  u        = e_{d/2-1}, the lowest-frequency rotate-half coordinate (RoPE barely
             rotates it over the context: theta^(-(d-2)/d) rad per position);
  level_j  = perm[j mod L], perm a seeded permutation of [0, L), L = 128 >= 2^(N-1)
             (selection compares tokens < 2^(N-1) apart: always distinct levels);
  k_j      = n_j (N(0,1), zero on u) + (level_j / 2) * u     -> exact in bf16;
  q_j      = 2 u + eps * n'_j,  eps = 0.25 (0.05 for the fp32 toy);
  v_j      ~ N(0, 1);
  passkey  (optional): keys of 5 consecutive positions at a seeded depth get
             k_j[u] = 128 (a salient block the cascade should retain).
Noise is drawn per chunk from torch.Generator(device).manual_seed(seed * 1_000_003 + start),
so a chunk is reproducible on its own; generating on the GPU and copying a chunk to
the host gives the oracle the identical bits.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

L_LEVELS = 128


@dataclass
class Synth:
    batch: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    seed: int
    eps: float = 0.25
    dtype: torch.dtype = torch.bfloat16
    passkey_depth: Optional[int] = None   # stream position of the 5-token passkey block

    def __post_init__(self):
        rs = np.random.RandomState(self.seed % (2 ** 31))
        self.perm = torch.from_numpy(rs.permutation(L_LEVELS).astype(np.float32))
        self.u = self.head_dim // 2 - 1

    def chunk(self, start: int, m: int, device="cpu"):
        """q [B,m,Hq,d], k/v [B,m,Hkv,d] for stream positions [start, start + m)."""
        B, Hq, Hk, d = self.batch, self.num_q_heads, self.num_kv_heads, self.head_dim
        gen = torch.Generator(device=device)
        gen.manual_seed(self.seed * 1_000_003 + start)
        f32 = torch.float32
        nk = torch.randn((B, m, Hk, d), generator=gen, device=device, dtype=f32)
        nq = torch.randn((B, m, Hq, d), generator=gen, device=device, dtype=f32)
        v = torch.randn((B, m, Hk, d), generator=gen, device=device, dtype=f32)
        pos = torch.arange(start, start + m, device=device)
        level = self.perm.to(device)[pos % L_LEVELS]                       # [m]
        k = nk.to(self.dtype).to(f32)
        k[..., self.u] = (level / 2.0)[None, :, None]
        if self.passkey_depth is not None:
            sel = (pos >= self.passkey_depth) & (pos < self.passkey_depth + 5)
            if bool(sel.any()):
                k[:, sel, :, self.u] = 128.0
        q = self.eps * nq
        q[..., self.u] = 2.0
        return q.to(self.dtype), k.to(self.dtype), v.to(self.dtype)


# BASELINE.json configs; seeds = 1_000_000 * k + 1000 * layer.
CONFIGS = {
    "cfg1_toy": dict(num_layers=1, batch=1, num_q_heads=1, num_kv_heads=1, head_dim=64, sink_size=4,
                     cache_size=64, num_cascades=4, stride=16, tokens=512, dtype="f32",
                     rope_theta=10000.0, eps=0.05),
    "cfg2_llama8b_4k": dict(num_layers=1, batch=1, num_q_heads=32, num_kv_heads=8, head_dim=128,
                            sink_size=64, cache_size=4096, num_cascades=4, stride=1024, tokens=32768,
                            dtype="bf16", rope_theta=500000.0, eps=0.25),
    "cfg3_1m_65k": dict(num_layers=1, batch=1, num_q_heads=32, num_kv_heads=8, head_dim=128,
                        sink_size=64, cache_size=65536, num_cascades=8, stride=4096, tokens=1 << 20,
                        dtype="bf16", rope_theta=500000.0, eps=0.25, passkey=True),
    "cfg4_decode": dict(num_layers=1, batch=64, num_q_heads=32, num_kv_heads=8, head_dim=128,
                        sink_size=64, cache_size=16384, num_cascades=4, stride=4096,
                        tokens=1 << 17, decode_steps=256, dtype="bf16", rope_theta=500000.0, eps=0.25),
    "cfg5_8gpu_32l": dict(num_layers=32, batch=1, num_q_heads=32, num_kv_heads=8, head_dim=128,
                          sink_size=64, cache_size=65536, num_cascades=8, stride=4096, tokens=1 << 20,
                          dtype="bf16", rope_theta=500000.0, eps=0.25, passkey=True),
}


def config_seed(k: int, layer: int = 0) -> int:
    return 1_000_000 * k + 1000 * layer


def passkey_depth(seed: int, tokens: int) -> int:
    rs = np.random.RandomState((seed + 17) % (2 ** 31))
    return int(rs.randint(tokens // 8, tokens - tokens // 8))
