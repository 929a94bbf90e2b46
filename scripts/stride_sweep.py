"""Stride sweep at 1M tokens (SURVEY §8(d) optional item; the B200 analogue of the paper's
Fig. 5c latency-vs-stride study).

The configs[2] workload (Llama-3-8B attention-layer shapes, 64 sinks + 8 x 8192 cascade,
2^20 synthetic tokens with a passkey block) is prefilled with strides m in {1024, 2048, 4096,
8192}.  One token stream is generated once on the device and sliced per stride; every call's
inputs are resident in HBM.  Per stride: one untimed pass, then one pass timed with CUDA
events; reported as tokens/s and ms per 1M tokens.

    python scripts/stride_sweep.py [--out profiles/stride_sweep_r01.json]
"""

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2406_17808_b200 import cascade as C  # noqa: E402
from paper_2406_17808_b200.synth import CONFIGS, Synth, config_seed, passkey_depth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--strides", default="1024,2048,4096,8192")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "stride_sweep_r01.json"))
    args = ap.parse_args()
    spec = dict(CONFIGS["cfg3_1m_65k"])
    T, Hq, Hk, d = spec["tokens"], spec["num_q_heads"], spec["num_kv_heads"], spec["head_dim"]
    seed = config_seed(3)
    syn = Synth(1, Hq, Hk, d, seed, eps=spec["eps"], passkey_depth=passkey_depth(seed, T))
    gen = 8192
    Q = torch.empty((T, Hq, d), dtype=torch.bfloat16, device="cuda")
    K = torch.empty((T, Hk, d), dtype=torch.bfloat16, device="cuda")
    V = torch.empty_like(K)
    for s in range(0, T, gen):
        q, k, v = syn.chunk(s, gen, device="cuda")
        Q[s:s + gen].copy_(q[0]); K[s:s + gen].copy_(k[0]); V[s:s + gen].copy_(v[0])
    O = torch.empty_like(Q)
    rows = []
    for m in [int(x) for x in args.strides.split(",")]:
        cfg = C.CascadeConfig(batch=1, num_q_heads=Hq, num_kv_heads=Hk, head_dim=d,
                              sink_size=spec["sink_size"], cache_size=spec["cache_size"],
                              num_cascades=spec["num_cascades"], max_stride=m, dtype="bf16",
                              rope_theta=spec["rope_theta"])
        cas = C.Cascade(cfg)

        def run():
            cas.reset(0)
            for s in range(0, T, m):
                cas.prefill_stride(0, Q[s:s + m].unsqueeze(0), K[s:s + m].unsqueeze(0),
                                   V[s:s + m].unsqueeze(0), out=O[s:s + m].unsqueeze(0))

        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        r = {"stride": m, "chunks": (T + m - 1) // m, "ms_per_1M": ms, "tok_per_s": T / (ms / 1e3),
             "n_cached_end": int(cas.state(0)["n_cached"])}
        rows.append(r)
        print(f"stride {m:5d}: {ms:8.1f} ms per 2^20 tokens, {r['tok_per_s'] / 1e3:7.1f}K tok/s", flush=True)
        cas.close()
    with open(args.out, "w") as f:
        json.dump({"workload": "configs[2] shape: 2^20 tokens, 64 sinks + 8 x 8192 cascade, 32q/8kv "
                               "d=128 bf16, one timed pass per stride after one untimed pass",
                   "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
