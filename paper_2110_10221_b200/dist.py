"""Sequence-sharded multi-GPU plumbing.

Sequences are independent, so each rank runs the one-GPU layer on a contiguous sequence range
chosen by `cora_shard_plan` (FLOP-balanced); the only exchange is the final all-gather of the
ragged outputs, done in place as one broadcast per rank (NCCL over NVLink on GPUs; gloo in the CPU
tests).  This module holds host bookkeeping and the collective call only -- no layer arithmetic.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

from .api import shard_plan


def shard_rows(lengths: Sequence[int], d_model: int, d_ff: int, world: int) -> Tuple[List[int], List[int]]:
    """(seq_begin[world+1], tok_begin[world+1]): rank r owns sequences [seq_begin[r], seq_begin[r+1])
    = packed rows [tok_begin[r], tok_begin[r+1])."""
    plan = shard_plan(list(lengths), d_model, d_ff, world)
    ro = [0]
    for L in lengths:
        ro.append(ro[-1] + int(L))
    return plan, [ro[b] for b in plan]


def allgather_ragged(y_full, y_local, tok_begin: Sequence[int], rank: int, world: int, group=None) -> None:
    """Gather every rank's packed rows into y_full[T, d] in original order (in place)."""
    import torch.distributed as dist

    if tok_begin[rank + 1] > tok_begin[rank]:
        y_full[tok_begin[rank]:tok_begin[rank + 1]].copy_(y_local)
    for r in range(world):
        if tok_begin[r + 1] > tok_begin[r]:
            dist.broadcast(y_full[tok_begin[r]:tok_begin[r + 1]], src=r, group=group)
