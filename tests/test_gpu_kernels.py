"""Focused GPU checks of kernel building blocks that parity runs might not stress."""
import numpy as np
import pytest
import torch

from paper_2406_17808_b200 import cascade as C

pytestmark = pytest.mark.gpu


def test_decode_scores_have_no_nan_and_sum_rule():
    """m = 1 leaves 127 masked query rows in every 128-row tile: their weight must be exactly
    ~0 (no NaN from the FMA-pipe exp2), and sum_j s_h[j] <= 1 - gamma (max over heads of rows
    that each sum to 1 - gamma)."""
    from paper_2406_17808_b200.synth import Synth
    cfg = C.CascadeConfig(batch=2, num_q_heads=4, num_kv_heads=1, head_dim=128, sink_size=4, cache_size=256,
                          num_cascades=2, max_stride=64, dtype="bf16", ema_gamma=0.99)
    gpu = C.Cascade(cfg)
    syn = Synth(2, 4, 1, 128, seed=3)
    q, k, v = syn.chunk(0, 64)
    gpu.prefill_stride(0, q.cuda(), k.cuda(), v.cuda())
    q, k, v = syn.chunk(64, 1)
    gpu.decode(0, q[:, 0].contiguous().cuda(), k[:, 0].contiguous().cuda(), v[:, 0].contiguous().cuda())
    s = gpu.last_scores(0).cpu().numpy()
    assert np.isfinite(s).all() and (s >= 0).all()
    tot = s.sum(-1)
    assert np.all(tot >= (1 - 0.99) * (1 - 1e-4)) and np.all(tot <= 4 * (1 - 0.99) * (1 + 1e-4))
