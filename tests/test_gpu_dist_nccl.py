"""Row a9 (the output gather) and the homogeneous policy's cross-rank reduction through NCCL on
the GPU.  gpurun has one GPU, so the process group has one rank: the collectives are the same
calls `bench.py` issues under torchrun (`all_gather_into_tensor` of each chunk's output shard on
a side stream; `all_reduce` of the score buffer between `cascade_attend` and `cascade_commit`),
and with one rank their results must equal the local data bit for bit.  The multi-rank host
logic (partition, gather layout, reduction) is covered by the world-size-2 gloo tests."""

import socket

import pytest
import torch
import torch.distributed as dist

from paper_2406_17808_b200 import cascade as C
from paper_2406_17808_b200.dist import gather_heads, homogeneous_step, shard_range
from paper_2406_17808_b200.synth import Synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_nccl_gather_of_output_shards_on_a_side_stream(nccl_group):
    """The bench's per-chunk gather: outputs of consecutive chunks all_gathered on a comm stream
    ordered after the compute stream by events; the gathered buffer (rank-major, no reshape copy)
    holds this rank's shard exactly."""
    q_sl, k_sl = shard_range(0, 1, 8, 2)
    cfg = C.CascadeConfig(batch=1, num_q_heads=8, num_kv_heads=2, head_dim=128, sink_size=4, cache_size=64,
                          num_cascades=4, max_stride=64, dtype="bf16")
    cas = C.Cascade(cfg)
    syn = Synth(1, 8, 2, 128, seed=77)
    comm = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    outs, gathered = [], []
    for c in range(4):
        q, k, v = (t.cuda() for t in syn.chunk(c * 64, 64))
        o = cas.prefill_stride(0, q[:, :, q_sl].contiguous(), k[:, :, k_sl].contiguous(), v[:, :, k_sl].contiguous())
        ev = torch.cuda.Event()
        ev.record(main)
        comm.wait_event(ev)
        with torch.cuda.stream(comm):
            buf = gather_heads(o, 1, assemble=False)
        outs.append(o)
        gathered.append(buf)
    torch.cuda.synchronize()
    for o, g in zip(outs, gathered):
        assert g.shape == (1,) + tuple(o.shape)
        assert torch.equal(g[0].view(torch.int16), o.view(torch.int16))
        assert torch.equal(gather_heads(o, 1).view(torch.int16), o.view(torch.int16))


def test_nccl_homogeneous_split_step_equals_single_call(nccl_group):
    """The homogeneous policy's split step with an NCCL all_reduce(MAX) of the score buffer (one
    rank: the reduction is the identity) equals the single-call step bit for bit, prefill and
    decode, and leaves the same cascade state."""
    cfg = C.CascadeConfig(batch=2, num_q_heads=8, num_kv_heads=2, head_dim=128, sink_size=4, cache_size=64,
                          num_cascades=4, max_stride=48, dtype="bf16", head_policy="homogeneous")
    a, b = C.Cascade(cfg), C.Cascade(cfg)
    syn = Synth(2, 8, 2, 128, seed=78)
    start = 0
    for m in (48, 48, 48, 31, 1, 1):
        q, k, v = (t.cuda() for t in syn.chunk(start, m))
        start += m
        o1 = a.prefill_stride(0, q, k, v) if m > 1 else \
            a.decode(0, q[:, 0].contiguous(), k[:, 0].contiguous(), v[:, 0].contiguous())[:, None]
        o2 = homogeneous_step(b, 0, q, k, v, reduce="max")
        torch.cuda.synchronize()
        assert torch.equal(o1.view(torch.int16), o2.view(torch.int16)), m
    sa, sb = a.state(0), b.state(0)
    for key in ("origin", "mu", "pe"):
        assert torch.equal(sa[key], sb[key]), key
