"""The split step (cascade_attend / cascade_score_buffer / cascade_commit) and checkpoint restore
(cascade_load_state), through the C ABI on one GPU."""

import numpy as np
import pytest
import torch

from paper_2406_17808_b200 import cascade as C
from paper_2406_17808_b200.dist import shard_range
from paper_2406_17808_b200.synth import Synth

pytestmark = pytest.mark.gpu


def _cfg(**kw):
    base = dict(batch=2, num_q_heads=16, num_kv_heads=4, head_dim=128, sink_size=8, cache_size=256,
                num_cascades=4, max_stride=128, dtype="bf16")
    base.update(kw)
    return C.CascadeConfig(**base)


@pytest.mark.parametrize("world", [2, 4])
def test_homogeneous_policy_under_kv_head_sharding(world):
    """Homogeneous heads with the kv-heads split over `world` shard handles on one device:
    attend on every shard, the element-wise MAX of the shards' score buffers (what the NCCL
    all_reduce(MAX) of dist.homogeneous_step computes across ranks) written back into each, then
    commit -- prefill chunks and decode steps give outputs, scores and cascade state bit-identical
    to one all-heads handle with the same policy."""
    full = C.Cascade(_cfg(head_policy="homogeneous"))
    Hq, Hkv = 16, 4
    shards = [C.Cascade(_cfg(num_q_heads=Hq // world, num_kv_heads=Hkv // world, head_policy="homogeneous"))
              for _ in range(world)]
    sl = [shard_range(r, world, Hq, Hkv) for r in range(world)]
    syn = Synth(2, Hq, Hkv, 128, seed=404)
    start = 0
    steps = [128, 128, 77, 128, 128, 1, 1, 1, 1, 1, 1]
    for m in steps:
        q, k, v = (t.cuda() for t in syn.chunk(start, m))
        start += m
        ref = full.prefill_stride(0, q, k, v) if m > 1 else \
            full.decode(0, q[:, 0].contiguous(), k[:, 0].contiguous(), v[:, 0].contiguous())[:, None]
        parts = []
        outs = []
        for r, (qs, ks) in enumerate(sl):
            qq, kk, vv = q[:, :, qs].contiguous(), k[:, :, ks].contiguous(), v[:, :, ks].contiguous()
            outs.append((shards[r].attend(0, qq, kk, vv), kk, vv))
            parts.append(shards[r].score_buffer(0))
        red = parts[0].clone()
        for p_ in parts[1:]:
            red = torch.maximum(red, p_)
        for r in range(world):
            parts[r].copy_(red[:, : parts[r].shape[1]])
            shards[r].commit(0, outs[r][1], outs[r][2])
        for r, (qs, _) in enumerate(sl):
            assert torch.equal(outs[r][0], ref[:, :, qs]), m
    torch.cuda.synchronize()
    st = full.state(0)
    for r, (_, ks) in enumerate(sl):
        sh = shards[r].state(0)
        for key in ("origin", "mu", "k", "v"):
            assert torch.equal(sh[key], st[key][:, ks]), key
        assert torch.equal(shards[r].last_scores(0), full.last_scores(0)[:, ks])


def test_split_step_equals_single_call_and_orders_calls():
    """attend + commit == prefill_stride / decode bit for bit (independent heads); between an attend
    and its commit every other call on that layer is refused (CASCADE_ERR_ORDER), other layers run."""
    cfg = _cfg(num_layers=2)
    a, b = C.Cascade(cfg), C.Cascade(cfg)
    syn = Synth(2, 16, 4, 128, seed=9)
    start = 0
    for m in [128, 128, 128, 128, 1, 1, 1]:
        q, k, v = (t.cuda() for t in syn.chunk(start, m))
        start += m
        o1 = a.prefill_stride(0, q, k, v) if m > 1 else \
            a.decode(0, q[:, 0].contiguous(), k[:, 0].contiguous(), v[:, 0].contiguous())[:, None]
        o2 = b.attend(0, q, k, v)
        with pytest.raises(C.CascadeError) as e:
            b.prefill_stride(0, q, k, v)
        assert e.value.code == -4
        with pytest.raises(C.CascadeError):
            b.state(0)
        b.prefill_stride(1, q, k, v)                        # another layer is free
        b.commit(0, k, v)
        assert torch.equal(o1, o2)
    torch.cuda.synchronize()
    sa, sb = a.state(0), b.state(0)
    for key in ("origin", "mu", "k", "v", "pe"):
        assert torch.equal(sa[key], sb[key]), key
    with pytest.raises(C.CascadeError):
        b.commit(0, k, v)                                   # nothing pending


def test_load_state_round_trip():
    """Checkpoint restore: a second handle loaded with the first's exported state (copied out)
    continues bit-identically through prefill chunks and decode steps; an unreachable mirror is
    refused."""
    cfg = _cfg()
    a, b = C.Cascade(cfg), C.Cascade(cfg)
    syn = Synth(2, 16, 4, 128, seed=17)
    start = 0
    for m in [128] * 5:
        a.prefill_stride(0, *(t.cuda() for t in syn.chunk(start, m)))
        start += m
    snap = {k_: (v_.clone() if torch.is_tensor(v_) else v_) for k_, v_ in a.state(0).items()}
    b.load_state(0, snap)
    for m in [128, 1, 1, 128, 1]:
        q, k, v = (t.cuda() for t in syn.chunk(start, m))
        start += m
        if m == 1:
            q, k, v = q[:, 0].contiguous(), k[:, 0].contiguous(), v[:, 0].contiguous()
            assert torch.equal(a.decode(0, q, k, v), b.decode(0, q, k, v))
        else:
            assert torch.equal(a.prefill_stride(0, q, k, v), b.prefill_stride(0, q, k, v))
    sa, sb = a.state(0), b.state(0)
    for key in ("origin", "mu", "k", "v", "pe"):
        assert torch.equal(sa[key], sb[key]), key
    bad = dict(snap)
    bad["xi"] = [1] + list(snap["xi"][1:])                  # sub-cache 1 not full: xi must be its count
    bad["counts"] = [3] + list(snap["counts"][1:])
    with pytest.raises(C.CascadeError):
        b.load_state(0, bad)


def test_misaligned_pointers_rejected_before_any_launch():
    """cascade.h: device I/O pointers must be 16-byte aligned (vector loads, TMA); a misaligned one
    is INVALID_ARG from the host check, with nothing launched and the mirror unchanged."""
    import ctypes
    cfg = _cfg(num_layers=1)
    cas = C.Cascade(cfg)
    syn = Synth(2, 16, 4, 128, seed=3)
    q, k, v = (t.cuda() for t in syn.chunk(0, 16))
    out = torch.empty_like(q)
    n0 = cas.launch_count()
    L = C.lib()
    bad = ctypes.c_void_p(q.data_ptr() + 2)
    rc = L.cascade_prefill_stride(cas._h, 0, bad, C._ptr(k), C._ptr(v), 16, C._ptr(out), C._stream(None))
    assert rc == -1
    rc = L.cascade_decode(cas._h, 0, C._ptr(q), ctypes.c_void_p(k.data_ptr() + 8), C._ptr(v), C._ptr(out),
                          C._stream(None))
    assert rc == -1
    assert cas.launch_count() == n0 and cas.state(0)["t"] == 0
    cas.prefill_stride(0, q, k, v)                      # the handle still works
    assert cas.state(0)["t"] == 16
