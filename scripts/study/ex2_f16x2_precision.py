"""Precision study for a next-round pass-1 option: evaluate the exp2 of the MUFU share with
`ex2.approx.f16x2` (two exp2 per MUFU op) -- the argument rounded to fp16, the result rounded
to fp16 -- instead of fp32 `ex2.approx`.  Emulated here in numpy on the synthetic recipe's
logits (configs[2] shapes, one kv-head, 4 q-heads x 128 query rows against 16K keys); reports
the max-abs O error (north-star bf16 tolerance 2e-2) and the LSE error, whose 2^(dLSE) - 1 is
the relative error it would put on every per-key mass of pass 2 (tolerance 1e-3).

    python scripts/study/ex2_f16x2_precision.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2406_17808_b200.synth import Synth  # noqa: E402


def main():
    n_keys, rows, d = 16384, 128, 128
    syn = Synth(1, 4, 1, d, seed=3, eps=0.25, dtype=torch.float32)
    _, k, v = syn.chunk(0, n_keys)
    q, _, _ = syn.chunk(n_keys, rows)
    K = k[0, :, 0].double().numpy()
    V = v[0, :, 0].double().numpy()
    scale_log2 = (1.0 / np.sqrt(d)) * np.log2(np.e)
    worst_o, worst_lse = 0.0, 0.0
    for h in range(4):
        Q = q[0, :, h].double().numpy()
        t = (Q @ K.T) * scale_log2                       # log2-domain logits
        m = t.max(axis=1, keepdims=True)
        x = t - m                                        # <= 0, as the kernel's exp2 argument
        p_ref = np.exp2(x)
        l_ref = p_ref.sum(axis=1)
        o_ref = (p_ref @ V) / l_ref[:, None]
        # 12 of 16 pairs on MUFU in f16x2 (argument and result in fp16), 4 of 16 exact-ish
        mufu = (np.arange(n_keys) // 2) % 16 < 12
        p16 = np.exp2(x.astype(np.float16).astype(np.float64)).astype(np.float16).astype(np.float64)
        p = np.where(mufu[None, :], p16, p_ref)
        p_bf16 = torch.from_numpy(p).to(torch.bfloat16).double().numpy()   # P operand of PV
        l = p.astype(np.float32).sum(axis=1, dtype=np.float64)
        o = (p_bf16 @ V) / l[:, None]
        worst_o = max(worst_o, float(np.abs(o - o_ref).max()))
        worst_lse = max(worst_lse, float(np.abs(np.log2(l) - np.log2(l_ref)).max()))
    print(f"max |dO| = {worst_o:.3e} (tolerance 2e-2);  max |dLSE2| = {worst_lse:.3e} "
          f"-> per-key mass rel. error up to {2 ** worst_lse - 1:.3e} (tolerance 1e-3)")


if __name__ == "__main__":
    main()
