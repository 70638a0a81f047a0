"""Utterance sharding across GPUs (one process per GPU, torch.distributed).

Rows of a decode batch are independent (model.hpp:89-91: row b of every
output depends only on row b of the inputs), so a large batch is split into
contiguous utterance ranges, each rank decodes its range on its own GPU with
its own decoder, and the hypotheses are gathered on the host of rank 0 by
utterance index.  There is no collective on the data path; the only
communication is the final host-side gather (gloo or NCCL object gather).
"""
from __future__ import annotations

from typing import Callable, List, Sequence


def shard_range(batch: int, rank: int, world: int) -> tuple:
    """Contiguous [b0, b1) utterance range of `rank` (balanced to +-1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return batch * rank // world, batch * (rank + 1) // world


def sort_by_length(out_len: Sequence[int]) -> List[int]:
    """Permutation putting longer utterances first so shards are balanced when
    lengths vary."""
    return sorted(range(len(out_len)), key=lambda b: -int(out_len[b]))


def decode_sharded(decode_fn: Callable, x, out_len, rank: int, world: int, group=None):
    """Decode this rank's utterance range with decode_fn(x_shard, len_shard)
    and gather every rank's hypotheses to rank 0 (None elsewhere)."""
    import torch.distributed as dist

    b0, b1 = shard_range(len(out_len), rank, world)
    local = decode_fn(x[b0:b1], out_len[b0:b1]) if b1 > b0 else []
    if world == 1:
        return list(local)
    gathered = [None] * world if rank == 0 else None
    dist.gather_object((b0, list(local)), gathered, dst=0, group=group)
    if rank != 0:
        return None
    out = [None] * len(out_len)
    for start, hyps in gathered:
        for i, h in enumerate(hyps):
            out[start + i] = h
    return out
