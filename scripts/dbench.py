"""Decode microbenchmark (configs[3] shape): fill by score injection, time single-token steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_17808_b200 import cascade as C
from paper_2406_17808_b200.synth import Synth

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 32
exact = len(sys.argv) > 3 and sys.argv[3] == "exact"
cfg = C.CascadeConfig(batch=B, num_q_heads=32, num_kv_heads=8, head_dim=128, sink_size=64, cache_size=16384,
                      num_cascades=4, max_stride=4096, dtype="bf16", exact_decode_rope=exact)
cas = C.Cascade(cfg)
syn = Synth(B, 32, 8, 128, seed=4)
g = torch.Generator(device="cuda").manual_seed(4)
for start in range(0, 1 << 15, 4096):
    _, k, v = syn.chunk(start, 4096, device="cuda")
    cas.update_with_scores(0, k, v, torch.rand((B, 8, cfg.s_tot + 4096), generator=g, device="cuda") * 1e-4)
qs = [syn.chunk((1 << 15) + i, 1, device="cuda") for i in range(steps)]
qs = [(q[:, 0].contiguous(), k[:, 0].contiguous(), v[:, 0].contiguous()) for q, k, v in qs]
out = torch.empty_like(qs[0][0])
for i in range(3):
    cas.decode(0, *qs[i], out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(3, steps):
    cas.decode(0, *qs[i], out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / (steps - 3)
n_c = cas.state(0)["n_cached"]
byt = B * 8 * (n_c + 1) * (4 * 128 + 20)   # K, V + mu r/w + s per key
print(f"{'exact' if exact else 'fast'} rope B={B} n_cached={n_c}: {ms:.3f} ms/step, {B / ms * 1e3:,.0f} tok/s, {byt / ms / 1e6:,.0f} GB/s algorithmic")
