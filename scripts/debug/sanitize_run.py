"""compute-sanitizer driver: a few strided-prefill chunks + decode steps through the C ABI.
    python scripts/debug/sanitize_run.py toy|cfg2|gqa [chunks]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2406_17808_b200 import cascade as C
from paper_2406_17808_b200.synth import Synth
which = sys.argv[1] if len(sys.argv) > 1 else "toy"
nchunks = int(sys.argv[2]) if len(sys.argv) > 2 else 4
if which == "toy":      # configs[0]: fp32 SIMT path
    cfg = C.CascadeConfig(batch=1, num_q_heads=1, num_kv_heads=1, head_dim=64, sink_size=4, cache_size=64,
                          num_cascades=4, max_stride=16, dtype="f32", rope_theta=10000.0)
    m = 16
elif which == "cfg2":   # configs[1] shape, bf16 tcgen05 path
    cfg = C.CascadeConfig(batch=1, num_q_heads=32, num_kv_heads=8, head_dim=128, sink_size=64, cache_size=4096,
                          num_cascades=4, max_stride=1024, dtype="bf16")
    m = 1024
else:                   # small bf16 with every kernel (fills, selections, decode), GQA 4
    cfg = C.CascadeConfig(batch=2, num_q_heads=8, num_kv_heads=2, head_dim=128, sink_size=4, cache_size=64,
                          num_cascades=4, max_stride=32, dtype="bf16")
    m = 32
cas = C.Cascade(cfg)
syn = Synth(cfg.batch, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, seed=3)
dt = cfg.torch_dtype
for c in range(nchunks):
    q, k, v = syn.chunk(c * m, m)
    cas.prefill_stride(0, q.to(dt).cuda(), k.to(dt).cuda(), v.to(dt).cuda())
for i in range(4):
    q, k, v = syn.chunk(nchunks * m + i, 1)
    cas.decode(0, q[:, 0].to(dt).contiguous().cuda(), k[:, 0].to(dt).contiguous().cuda(),
               v[:, 0].to(dt).contiguous().cuda())
torch.cuda.synchronize()
st = cas.state(0)
print(which, "ok: n_cached", st["n_cached"], "launches", cas.launch_count())
