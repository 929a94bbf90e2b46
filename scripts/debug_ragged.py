"""Debug helper: ragged bf16 chunks through the C ABI vs the oracle, per-row error summary.
Usage: debug_ragged.py <head_dim>"""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2406_17808_b200 import cascade as C
from paper_2406_17808_b200.synth import Synth
from oracle.model import CascadeOracle, OracleConfig
d = int(sys.argv[1])
cfg = C.CascadeConfig(batch=2, num_q_heads=4, num_kv_heads=2, head_dim=d, sink_size=5, cache_size=384,
                      num_cascades=3, max_stride=300, dtype="bf16")
syn = Synth(2, 4, 2, d, seed=200 + d)
gpu = C.Cascade(cfg)
orc = CascadeOracle(OracleConfig(1, 2, 4, 2, d, 5, 384, 3, gamma=cfg.ema_gamma, rope_theta=cfg.rope_theta, round_operands="bf16"))
f64 = lambda t: t.to(torch.float64).cpu().numpy()
start = 0
for m in [200, 77]:
    q, k, v = syn.chunk(start, m); start += m
    out = gpu.prefill_stride(0, q.cuda(), k.cuda(), v.cuda())
    ref, _ = orc.prefill_stride(0, f64(q), f64(k), f64(v))
    err = np.abs(f64(out) - ref)   # [B, m, Hq, d]
    e = err.max(axis=-1)
    print("m", m, "max", err.max(), "rows>0.02:", int((e > 0.02).sum()), "of", e.size)
    bad = np.argwhere(e > 0.02)[:10]
    print(bad)
