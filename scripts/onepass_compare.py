"""The paper's one-pass mass estimator (Alg. 3's normaliser l + l rho / gamma, P:646;
CASCADE_OPT_ONEPASS_SCORES) against the exact two-pass mass (reading Q6), through the CUDA path,
on the same synthetic passkey streams (Llama-3-8B attention shape, 64 sinks, stride 4096):

  * the per-key mass of the first chunks, while both caches still hold the same tokens:
    relative deviation of the estimate from the exact mass (all keys, and the top-1 % by mass);
  * the cache after the whole stream: passkey tokens kept (of 5, per kv-head), the share of
    resident origins the two modes have in common, and mu of the common residents;
  * prefill throughput of both modes (the estimate has no second pass).

    python scripts/onepass_compare.py [--tokens 262144] [--cache 16384] [--out profiles/r02/onepass_compare.json]
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


def run(mode, N, tokens, cache, depth, stride=4096, seed=4242, keep_chunks=2):
    cfg = C.CascadeConfig(batch=1, num_q_heads=32, num_kv_heads=8, head_dim=128, sink_size=64,
                          cache_size=cache, num_cascades=N, max_stride=stride, dtype="bf16",
                          rope_theta=500000.0, score_mode=mode)
    syn = Synth(1, 32, 8, 128, seed=seed, passkey_depth=depth)
    cas = C.Cascade(cfg)
    early = []
    torch.cuda.synchronize()
    t0 = time.time()
    for i, start in enumerate(range(0, tokens, stride)):
        q, k, v = syn.chunk(start, min(stride, tokens - start), device="cuda")
        cas.prefill_stride(0, q, k, v)
        if i < keep_chunks:
            early.append(cas.last_scores(0).cpu().numpy())
    torch.cuda.synchronize()
    dt = time.time() - t0
    st = cas.state(0)
    out = dict(origin=st["origin"].cpu().numpy()[0], mu=st["mu"].cpu().numpy()[0], early=early, secs=dt)
    cas.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=1 << 18)
    ap.add_argument("--cache", type=int, default=16384)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "onepass_compare.json"))
    a = ap.parse_args()
    res = []
    for N in (4, 8):
        depth = a.tokens // 3
        ex = run("exact", N, a.tokens, a.cache, depth)
        op = run("onepass", N, a.tokens, a.cache, depth)
        dev_all, dev_top = [], []
        for se, so in zip(ex["early"], op["early"]):
            m = se > 0
            r = np.abs(so[m] - se[m]) / se[m]
            dev_all.append(float(np.median(r)))
            thr = np.quantile(se[m], 0.99)
            dev_top.append(float(np.median(np.abs(so[se >= thr] - se[se >= thr]) / se[se >= thr])))
        keys = np.arange(depth, depth + 5)
        kept = lambda org: [int(np.isin(keys, org[g]).sum()) for g in range(org.shape[0])]
        common, mu_rel = [], []
        for g in range(ex["origin"].shape[0]):
            oe, oo = ex["origin"][g], op["origin"][g]
            se_, so_ = set(oe[oe >= 0].tolist()), set(oo[oo >= 0].tolist())
            common.append(len(se_ & so_) / max(1, len(se_)))
            pos_e = {o: i for i, o in enumerate(oe) if o >= 0}
            pos_o = {o: i for i, o in enumerate(oo) if o >= 0}
            both = [o for o in se_ & so_]
            me = np.array([ex["mu"][g, pos_e[o]] for o in both])
            mo = np.array([op["mu"][g, pos_o[o]] for o in both])
            ok = me > 0
            mu_rel.append(float(np.median(np.abs(mo[ok] - me[ok]) / me[ok])) if ok.any() else None)
        row = {"N": N, "tokens": a.tokens, "cache": a.cache, "passkey_depth": depth,
               "early_chunk_mass_median_rel_dev_all_keys": dev_all,
               "early_chunk_mass_median_rel_dev_top1pct_keys": dev_top,
               "passkey_kept_exact": kept(ex["origin"]), "passkey_kept_onepass": kept(op["origin"]),
               "resident_origins_in_common": float(np.mean(common)),
               "mu_common_residents_median_rel_dev": mu_rel,
               "prefill_secs_exact": ex["secs"], "prefill_secs_onepass": op["secs"]}
        print(json.dumps(row), flush=True)
        res.append(row)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
