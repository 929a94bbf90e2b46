"""World-size-2 gloo test (CPU) of the head-sharded multi-GPU path's host logic.

Each rank runs the (CPU, test-only) oracle on its shard of kv-heads and q-heads exactly as
bench.py shards them for the GPU path, then the outputs are gathered with
`paper_2406_17808_b200.dist.gather_heads`; the gathered output and each rank's cascade state
must equal a single-process run over all heads (independent head policy)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.model import CascadeOracle, OracleConfig
    from paper_2406_17808_b200.dist import gather_heads, shard_range
    from paper_2406_17808_b200.synth import Synth

    B, Hq, Hkv, d, m = 2, 8, 4, 16, 6
    syn = Synth(B, Hq, Hkv, d, seed=21, dtype=torch.float32)
    qs, ks = shard_range(rank, world, Hq, Hkv)
    cfg = OracleConfig(1, B, Hq // world, Hkv // world, d, 2, 8, 2, gamma=0.9)
    orc = CascadeOracle(cfg)
    outs = []
    for start in range(0, 5 * m, m):
        q, k, v = syn.chunk(start, m)
        o, _ = orc.prefill_stride(0, q[:, :, qs].double().numpy(), k[:, :, ks].double().numpy(),
                                  v[:, :, ks].double().numpy())
        full = gather_heads(torch.from_numpy(o), world)
        outs.append(full.numpy())
    st = orc.state(0)
    gathered = [None] * world
    dist.all_gather_object(gathered, st["origin"])
    if rank == 0:
        result_q.put((np.stack(outs), np.concatenate(gathered, axis=1)))
    dist.barrier()
    dist.destroy_process_group()


def test_head_sharded_prefill_equals_single_process():
    from oracle.model import CascadeOracle, OracleConfig
    from paper_2406_17808_b200.synth import Synth

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs, origins = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0

    B, Hq, Hkv, d, m = 2, 8, 4, 16, 6
    syn = Synth(B, Hq, Hkv, d, seed=21, dtype=torch.float32)
    orc = CascadeOracle(OracleConfig(1, B, Hq, Hkv, d, 2, 8, 2, gamma=0.9))
    ref = []
    for start in range(0, 5 * m, m):
        qq, kk, vv = syn.chunk(start, m)
        o, _ = orc.prefill_stride(0, qq.double().numpy(), kk.double().numpy(), vv.double().numpy())
        ref.append(o)
    np.testing.assert_array_equal(outs, np.stack(ref))
    np.testing.assert_array_equal(origins, orc.state(0)["origin"])


def test_shard_range_rejects_uneven_split():
    from paper_2406_17808_b200.dist import shard_range
    assert shard_range(1, 4, 32, 8) == (slice(8, 16), slice(2, 4))
    with pytest.raises(ValueError):
        shard_range(0, 3, 32, 8)


def _homog_worker(rank, world, port, result_q):
    """Rank r computes its kv-head shard's per-key masses with the oracle (independent policy,
    max over each GQA group), reduces them over its local kv-heads, then all_reduce(MAX) over the
    ranks -- the reduction dist.homogeneous_step applies to the library's score buffer."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.model import CascadeOracle, OracleConfig
    from paper_2406_17808_b200.dist import shard_range
    from paper_2406_17808_b200.synth import Synth
    B, Hq, Hkv, d, m = 1, 8, 4, 16, 6
    syn = Synth(B, Hq, Hkv, d, seed=33, dtype=torch.float32)
    qs, ks = shard_range(rank, world, Hq, Hkv)
    orc = CascadeOracle(OracleConfig(1, B, Hq // world, Hkv // world, d, 2, 8, 2, gamma=0.9))
    q, k, v = syn.chunk(0, m)
    _, s = orc.prefill_stride(0, q[:, :, qs].double().numpy(), k[:, :, ks].double().numpy(),
                              v[:, :, ks].double().numpy())
    local = torch.from_numpy(s.max(axis=1))                 # [B, S_tot + m]: max over local kv-heads
    dist.all_reduce(local, op=dist.ReduceOp.MAX)
    if rank == 0:
        result_q.put(local.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_homogeneous_reduction_across_ranks_is_the_all_heads_max():
    from oracle.model import CascadeOracle, OracleConfig
    from paper_2406_17808_b200.synth import Synth
    world = 2
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_homog_worker, args=(r, world, port, q_)) for r in range(world)]
    for p in procs:
        p.start()
    got = q_.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    B, Hq, Hkv, d, m = 1, 8, 4, 16, 6
    syn = Synth(B, Hq, Hkv, d, seed=33, dtype=torch.float32)
    hom = CascadeOracle(OracleConfig(1, B, Hq, Hkv, d, 2, 8, 2, gamma=0.9, head_policy="homogeneous"))
    q, k, v = syn.chunk(0, m)
    _, s = hom.prefill_stride(0, q.double().numpy(), k.double().numpy(), v.double().numpy())
    np.testing.assert_array_equal(got, s[:, 0])
