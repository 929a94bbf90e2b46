"""Steady-state kernel microbenchmark: fill the cascade by score injection up to a target
occupancy, then time K prefill chunks and report each kernel class (CUDA events on the
launch stream, via cascade_profile_*).  Usage: kbench.py [fill_chunks] [timed_chunks] [m]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_17808_b200 import cascade as C
from paper_2406_17808_b200.synth import Synth

fill = int(sys.argv[1]) if len(sys.argv) > 1 else 200
timed = int(sys.argv[2]) if len(sys.argv) > 2 else 5
m = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
mode = sys.argv[4] if len(sys.argv) > 4 else "exact"      # or "onepass"
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["bf16_tflops"]
cfg = C.CascadeConfig(batch=1, num_q_heads=32, num_kv_heads=8, head_dim=128, sink_size=64, cache_size=65536,
                      num_cascades=8, max_stride=m, dtype="bf16", score_mode=mode)
cas = C.Cascade(cfg)
syn = Synth(1, 32, 8, 128, seed=11)
g = torch.Generator(device="cuda").manual_seed(1)
for c in range(fill):
    _, k, v = syn.chunk(c * m, m, device="cuda")
    s = torch.rand((1, 8, cfg.s_tot + m), generator=g, device="cuda") * 1e-4
    cas.update_with_scores(0, k, v, s)
qs = [syn.chunk((fill + c) * m, m, device="cuda") for c in range(timed + 2)]
for c in range(2):
    cas.prefill_stride(0, *qs[c])
torch.cuda.synchronize()
cas.profile_enable(True); cas.profile_read()
for c in range(2, timed + 2):
    cas.prefill_stride(0, *qs[c])
torch.cuda.synchronize()
pr = cas.profile_read()
n_c = cas.state(0)["n_cached"]
print(f"n_cached after: {n_c}")
for k, (ms, cnt, work) in pr.items():
    if not cnt: continue
    per = ms / cnt
    if k in ("attn_fwd", "attn_score"):
        tf = work / (ms / 1e3) / 1e12
        print(f"{k:12s} {per:7.3f} ms/chunk  {tf:7.1f} TFLOP/s useful  ({tf/peak*100:5.1f}% of {peak})")
    else:
        print(f"{k:12s} {per:7.3f} ms/chunk  {work/(ms/1e3)/1e9:7.1f} GB/s algorithmic")
tot = sum(v[0] for v in pr.values()) / timed
print(f"total {tot:.3f} ms/chunk -> {m / (tot / 1e3):,.0f} tok/s at this occupancy")
