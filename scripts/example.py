"""Minimal end-to-end use of the library: a strided prefill of a synthetic sequence through a
cascade, a few decode steps, and the exported cache state.

    python scripts/example.py            (needs a B200 and the built library)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2406_17808_b200 import Cascade, CascadeConfig
from paper_2406_17808_b200.synth import Synth

cfg = CascadeConfig(batch=1, num_q_heads=32, num_kv_heads=8, head_dim=128, sink_size=64,
                    cache_size=4096, num_cascades=4, max_stride=1024, dtype="bf16")
cas = Cascade(cfg)                                   # workspace on cuda:0, every cascade empty
syn = Synth(1, 32, 8, 128, seed=0)
for start in range(0, 16384, 1024):                  # Alg. 1: one call per 1024-token chunk
    q, k, v = syn.chunk(start, 1024, device="cuda")  # [B, m, H, d] bf16, keys pre-RoPE
    out = cas.prefill_stride(0, q, k, v)             # attention over [sinks | cascade | chunk]
for t in range(4):                                   # single-token decode (Eq. 2) + update
    q, k, v = syn.chunk(16384 + t, 1, device="cuda")
    o = cas.decode(0, q[:, 0].contiguous(), k[:, 0].contiguous(), v[:, 0].contiguous())
st = cas.state(0)
print(f"tokens seen {st['t']}, resident {st['n_cached']} (sinks {st['sink_count']}, "
      f"sub-caches {st['counts']}), output {tuple(o.shape)} {o.dtype}")
torch.cuda.synchronize()
