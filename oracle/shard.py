"""Sequence-sharded multi-GPU partition (TEST INFRASTRUCTURE ONLY).

BASELINE.json north_star: "The batch is partitioned across the 8 GPUs of one
box by sequence, balanced on sum(L_i d + L_i^2) FLOPs."  The per-sequence cost
is the exact useful FLOP count of that sequence (oracle/flops.py with B = 1):
    cost(L) = 2 L (4 d^2 + 2 d d_ff) + 4 d L^2.
Reading s1: ranks own CONTIGUOUS sequence ranges (so outputs land
in order with no permutation); the plan minimises the maximum rank cost C*,
and among optimal plans the canonical one is greedy-left: rank r takes
sequences while its running cost stays <= C*.
"""
from __future__ import annotations

from functools import lru_cache
from typing import List, Sequence


def shard_cost(L: int, d: int, d_ff: int) -> int:
    L = int(L)
    return 2 * L * (4 * d * d + 2 * d * d_ff) + 4 * d * L * L


def _optimal_capacity(costs: Sequence[int], n_ranks: int) -> int:
    """min over contiguous partitions into <= n_ranks parts of the max part cost (plain DP)."""
    B = len(costs)

    @lru_cache(maxsize=None)
    def best(i: int, r: int) -> int:
        # best max-cost for costs[i:] using at most r parts
        if i == B:
            return 0
        if r == 0:
            return 1 << 62
        out = 1 << 62
        run = 0
        for j in range(i, B):
            run += costs[j]
            out = min(out, max(run, best(j + 1, r - 1)))
        return out

    return best(0, n_ranks)


def shard_plan(lengths: Sequence[int], d: int, d_ff: int, n_ranks: int) -> List[int]:
    """seq_begin[0..n_ranks]: rank r owns sequences [seq_begin[r], seq_begin[r+1])."""
    costs = [shard_cost(L, d, d_ff) for L in lengths]
    B = len(costs)
    cap = _optimal_capacity(tuple(costs), n_ranks) if B else 0
    begin = [0]
    i = 0
    for _r in range(n_ranks - 1):
        run = 0
        while i < B and run + costs[i] <= cap:
            run += costs[i]
            i += 1
        begin.append(i)
    begin.append(B)
    return begin
