"""Runs a few prefill chunks with a sync after each, printing timings (debug harness)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_17808_b200 import cascade as C
from paper_2406_17808_b200.synth import Synth

m = int(sys.argv[1]); nch = int(sys.argv[2]); Hq = int(sys.argv[3]); Hkv = int(sys.argv[4])
cache = int(sys.argv[5]) if len(sys.argv) > 5 else 65536
N = int(sys.argv[6]) if len(sys.argv) > 6 else 8
cfg = C.CascadeConfig(batch=1, num_q_heads=Hq, num_kv_heads=Hkv, head_dim=128, sink_size=64,
                      cache_size=cache, num_cascades=N, max_stride=m, dtype="bf16")
cas = C.Cascade(cfg)
syn = Synth(1, Hq, Hkv, 128, seed=3)
cas.profile_enable(True)
for c in range(nch):
    q, k, v = syn.chunk(c * m, m, device="cuda")
    t0 = time.time()
    out = cas.prefill_stride(0, q, k, v)
    torch.cuda.synchronize()
    pr = cas.profile_read()
    print(f"chunk {c}: {1e3*(time.time()-t0):.1f} ms  " + " ".join(f"{k}={v[0]:.2f}" for k, v in pr.items() if v[1]), flush=True)
print("ok", float(out.float().abs().mean()))
