"""Sequence-sharded multi-GPU partition (TEST INFRASTRUCTURE ONLY).

BASELINE.json north_star: "The batch is partitioned across the 8 GPUs of one
box by sequence, balanced on sum(L_i d + L_i^2) FLOPs."  The per-sequence cost
is the exact useful FLOP count of that sequence (oracle/flops.py with B = 1):
    cost(L) = 2 L (4 d^2 + 2 d d_ff) + 4 d L^2.
Reading s1: ranks own CONTIGUOUS sequence ranges (so outputs land
in order with no permutation); the plan minimises the maximum rank cost C*,
and among optimal plans the canonical one is greedy-left: rank r takes
sequences while its running cost stays <= C*.
Reading s2: when the batch is packed into short-sequence windows
(reading f4-r1; batches of <= PACK_MAX_BATCH sequences), a cut never splits a
window, so every rank rebuilds exactly the one-GPU windows of its sequences
(the G-rank result is then the one-GPU result row for row).  The cut
positions allowed are those no window spans; the plan is optimal and
greedy-left over them.
"""
from __future__ import annotations

from functools import lru_cache
from typing import List, Sequence

from .layout import short_windows

PACK_MAX_BATCH = 1024  # reading f4-r1: windows are built for batches of at most this many sequences


def shard_cost(L: int, d: int, d_ff: int) -> int:
    L = int(L)
    return 2 * L * (4 * d * d + 2 * d * d_ff) + 4 * d * L * L


def allowed_cuts(lengths: Sequence[int]) -> List[bool]:
    """allowed[c] for c in 0..B: may a rank boundary fall before sequence c?  (reading s2)
    Forbidden inside a short-sequence window: between its first and its last member."""
    B = len(lengths)
    ok = [True] * (B + 1)
    if B > PACK_MAX_BATCH:
        return ok
    for b0, _w, ns in short_windows(lengths):
        members = [b for b in range(b0, B) if 0 < int(lengths[b])][:ns]
        for c in range(b0 + 1, members[-1] + 1):
            ok[c] = False
    return ok


def _optimal_capacity(costs: Sequence[int], n_ranks: int, ok: Sequence[bool]) -> int:
    """min over contiguous partitions into <= n_ranks parts, cut only where ok, of the max part cost (DP)."""
    B = len(costs)

    @lru_cache(maxsize=None)
    def best(i: int, r: int) -> int:
        # best max-cost for costs[i:] using at most r parts (a part may end at j + 1 only if ok[j + 1])
        if i == B:
            return 0
        if r == 0:
            return 1 << 62
        out = 1 << 62
        run = 0
        for j in range(i, B):
            run += costs[j]
            if ok[j + 1]:
                out = min(out, max(run, best(j + 1, r - 1)))
        return out

    return best(0, n_ranks)


def shard_plan(lengths: Sequence[int], d: int, d_ff: int, n_ranks: int) -> List[int]:
    """seq_begin[0..n_ranks]: rank r owns sequences [seq_begin[r], seq_begin[r+1]) (readings s1, s2)."""
    costs = [shard_cost(L, d, d_ff) for L in lengths]
    ok = allowed_cuts(lengths)
    B = len(costs)
    cap = _optimal_capacity(tuple(costs), n_ranks, tuple(ok)) if B else 0
    begin = [0]
    i = 0
    for _r in range(n_ranks - 1):
        # greedy-left: the furthest allowed cut whose part stays <= cap
        run, j, last = 0, i, i
        while j < B and run + costs[j] <= cap:
            run += costs[j]
            j += 1
            if ok[j]:
                last = j
        i = last
        begin.append(i)
    begin.append(B)
    return begin
