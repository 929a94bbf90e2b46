"""Head sharding across GPUs (row a9 of SURVEY.md section 8) -- plumbing only.

The cascades of different kv-heads are independent under the paper's independent head
policy: every (layer, sequence, kv-head) keeps its own sink buffer, sub-caches and
EMA scores, and token selection never looks across heads.  So N ranks split the kv-heads
(and their G = Hq / Hkv query heads) with no exchange of cascade state; the only collective
is gathering the attention outputs of a chunk (NCCL all_gather over NVLink, one call per
chunk on a side stream).

Layout: rank r owns kv-heads [r*Hkv/N, (r+1)*Hkv/N) and q-heads [r*Hq/N, (r+1)*Hq/N) (the q
heads of a GQA group are contiguous).  A rank's output shard is [B, m, Hq/N, d];
`gather_heads` all_gathers the shards into [N, B, m, Hq/N, d] and returns the
[B, m, Hq, d] view in head order.
"""

from __future__ import annotations

from typing import Tuple

import torch
import torch.distributed as dist


def shard_range(rank: int, world: int, num_q_heads: int, num_kv_heads: int) -> Tuple[slice, slice]:
    """(q-head slice, kv-head slice) owned by `rank`."""
    if num_kv_heads % world:
        raise ValueError(f"{num_kv_heads} kv-heads do not split across {world} ranks")
    hk = num_kv_heads // world
    hq = num_q_heads // world
    return slice(rank * hq, (rank + 1) * hq), slice(rank * hk, (rank + 1) * hk)


def gather_heads(out_shard: torch.Tensor, world: int, buf: torch.Tensor | None = None,
                 group=None, assemble: bool = True) -> torch.Tensor:
    """all_gather [B, m, Hq/N, d] shards into buf [N, B, m, Hq/N, d].

    assemble=True returns the [B, m, Hq, d] tensor in head order (a copy: the gathered layout is
    rank-major); assemble=False returns the gather buffer itself (no copy), which is what the
    benchmark's per-chunk gather uses."""
    B, m, hq, d = out_shard.shape
    if buf is None:
        buf = torch.empty((world, B, m, hq, d), dtype=out_shard.dtype, device=out_shard.device)
    dist.all_gather_into_tensor(buf.view(-1), out_shard.contiguous().view(-1), group=group)
    if not assemble:
        return buf
    return buf.permute(1, 2, 0, 3, 4).reshape(B, m, world * hq, d)


def homogeneous_step(cas, layer: int, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                     out: torch.Tensor | None = None, group=None, reduce: str = "max", stream=None) -> torch.Tensor:
    """One Alg. 1 step under the homogeneous head policy with kv-head sharding.

    Homogeneous heads take ONE selection decision per sequence from s reduced over all kv-heads,
    which now live on different ranks: the library's split step computes the attention and the
    per-key mass reduced over the LOCAL kv-heads (cascade_attend), the ranks reduce that score
    buffer in place with an all_reduce (max; mean = sum of the equal-sized local means / world),
    and cascade_commit folds the global s and inserts the chunk.  m = 1 (q [B, 1, Hq/N, d]) is a
    decode step."""
    out = cas.attend(layer, q, k, v, out=out, stream=stream)
    s = cas.score_buffer(layer)
    with torch.cuda.stream(stream) if stream is not None else _null():
        if reduce == "max":
            dist.all_reduce(s, op=dist.ReduceOp.MAX, group=group)
        elif reduce == "mean":
            dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
            s.div_(dist.get_world_size(group))
        else:
            raise ValueError(reduce)
    cas.commit(layer, k, v, stream=stream)
    return out


class _null:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False
