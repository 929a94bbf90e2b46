"""Synthetic retention sweep (the mechanism of the paper's passkey
experiments, and of Eq. 4), run through the CUDA path.

For N in {1, 2, 4, 8, 16} sub-caches, with and without token selection (Q3), one sequence of
Llama-3-8B attention-layer shapes (32 q / 8 kv heads, d = 128, bf16) streams through a
64-sink + 16K cascade in 4096-token chunks, with a 5-token passkey block (salient keys,
DESIGN.md "Input recipe") planted at a given depth.  Reported per configuration, from the
exported cache state after the last chunk:
  * passkey tokens still resident, averaged over the 8 kv-heads (of 5);
  * the window span (newest - oldest non-sink origin + 1) against Eq. 4's S~ = c (2^N - 1);
  * residents and the share of the stream they stand for.

    python scripts/retention_sweep.py [--tokens 131072] [--out profiles/retention_sweep_r01.json]
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2406_17808_b200 import cascade as C  # noqa: E402
from paper_2406_17808_b200.synth import Synth  # noqa: E402


def run(N, selection, tokens, depth, cache=16384, stride=4096, seed=4242):
    cfg = C.CascadeConfig(batch=1, num_q_heads=32, num_kv_heads=8, head_dim=128, sink_size=64,
                          cache_size=cache, num_cascades=N, max_stride=stride, dtype="bf16",
                          rope_theta=500000.0, selection=selection)
    syn = Synth(1, 32, 8, 128, seed=seed, passkey_depth=depth)
    cas = C.Cascade(cfg)
    for start in range(0, tokens, stride):
        q, k, v = syn.chunk(start, min(stride, tokens - start), device="cuda")
        cas.prefill_stride(0, q, k, v)
    torch.cuda.synchronize()
    st = cas.state(0)
    org = st["origin"].cpu().numpy()[0]                      # [Hkv, S_tot]
    cas.close()
    keys = np.arange(depth, depth + 5)
    kept = [int(np.isin(keys, org[g]).sum()) for g in range(org.shape[0])]
    spans = []
    for g in range(org.shape[0]):
        o = org[g, 64:]
        o = o[o >= 0]
        spans.append(int(o.max() - o.min() + 1) if o.size else 0)
    c = cache // N
    return {"N": N, "selection": selection, "depth": depth, "passkey_kept_mean": float(np.mean(kept)),
            "passkey_kept_per_head": kept, "span_max": max(spans), "span_min": min(spans),
            "eq4_span": c * (2 ** N - 1), "n_cached": int(st["n_cached"]), "tokens": tokens}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=131072)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "retention_sweep_r01.json"))
    args = ap.parse_args()
    rows = []
    t0 = time.time()
    for frac in (0.25, 0.75):
        depth = int(args.tokens * frac) + 1000
        for N in (1, 2, 4, 8, 16):
            for sel in (True, False):
                r = run(N, sel, args.tokens, depth)
                rows.append(r)
                print(f"depth {depth:6d}  N={N:2d}  selection={'on ' if sel else 'off'}  passkey kept "
                      f"{r['passkey_kept_mean']:.2f}/5  span {r['span_min']}-{r['span_max']} "
                      f"(Eq. 4: {r['eq4_span']})  residents {r['n_cached']}", flush=True)
    with open(args.out, "w") as f:
        json.dump({"tokens": args.tokens, "cache": 16384, "sinks": 64, "stride": 4096,
                   "heads": "32q/8kv d=128 bf16", "seconds": time.time() - t0, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
