"""Pins for oracle/flops.py (instrumented loops, SPEC example) and oracle/shard.py (exhaustive search)."""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_spec_qkt_macs():
    for ex in GOLD["qkt_macs"]:
        assert oracle.qkt_macs(ex["lengths"], ex["heads"], ex["head_dim"]) == ex["ragged"], ex["cite"]
        assert oracle.qkt_macs(ex["lengths"], ex["heads"], ex["head_dim"], pad_to=max(ex["lengths"])) == ex["padded"]


@pytest.mark.parametrize("lengths,d,H,dff", [([3, 7, 1, 5], 16, 2, 32), ([2, 4], 8, 1, 8), ([0, 9, 4], 12, 3, 20)])
def test_closed_form_equals_instrumented_loops(lengths, d, H, dff):
    assert oracle.useful_flops(lengths, d, dff) == 2 * oracle.useful_macs_bruteforce(lengths, d, H, dff)
    assert oracle.padded_flops(lengths, d, dff) == 2 * oracle.padded_macs_bruteforce(lengths, d, H, dff)
    assert oracle.padded_flops(lengths, d, dff, pad_to=11) == 2 * oracle.padded_macs_bruteforce(lengths, d, H, dff, 11)


def test_c1_flop_numbers():
    # C1 useful 70 912 FLOP, padded-to-batch-max 127 232.
    L, d, H, dff = synth.config("C1")
    assert oracle.useful_flops(L, d, dff) == 70912
    assert oracle.padded_flops(L, d, dff) == 127232


def test_ratio_one_iff_equal_lengths():
    assert oracle.padded_flops([64] * 5, 512, 2048) == oracle.useful_flops([64] * 5, 512, 2048)
    rng = np.random.default_rng(0)
    for _ in range(20):
        L = list(rng.integers(1, 512, size=8))
        if len(set(L)) > 1:
            assert oracle.padded_flops(L, 512, 2048) > oracle.useful_flops(L, 512, 2048)


def _all_partitions(B, R):
    """Every way to cut range(B) into R contiguous (possibly empty) parts -> seq_begin lists."""
    for cuts in itertools.combinations_with_replacement(range(B + 1), R - 1):
        yield [0, *cuts, B]


def _windows_split_at(lengths, c):
    """The short-sequence windows of the two sub-batches [0, c) and [c, B), in global sequence indices."""
    left = oracle.short_windows(lengths[:c])
    right = [(b0 + c, w, ns) for b0, w, ns in oracle.short_windows(lengths[c:])]
    return left + right


@pytest.mark.parametrize("seed", range(8))
def test_allowed_cuts_are_exactly_the_window_preserving_cuts(seed):
    # reading s2: a cut is allowed iff the two sides rebuild exactly the one-GPU windows (f4-r1)
    rng = np.random.default_rng(100 + seed)
    B = int(rng.integers(1, 30))
    L = [int(x) for x in rng.choice([0, 1, 5, 30, 64, 100, 128, 129, 300], size=B)]
    ok = oracle.shard.allowed_cuts(L)
    whole = oracle.short_windows(L)
    assert ok[0] and ok[B]
    for c in range(1, B):
        assert ok[c] == (_windows_split_at(L, c) == whole), (L, c)


def test_allowed_cuts_unconstrained_above_pack_limit():
    L = [5] * (oracle.shard.PACK_MAX_BATCH + 1)  # no windows are built for this batch
    assert all(oracle.shard.allowed_cuts(L))


@pytest.mark.parametrize("seed", range(8))
def test_shard_plan_is_optimal_and_canonical(seed):
    rng = np.random.default_rng(seed)
    B, R = int(rng.integers(1, 9)), int(rng.integers(1, 5))
    L = [int(x) for x in rng.choice([0, 3, 40, 100, 200, 350, 512], size=B)]
    d, dff = 512, 2048
    cost = [oracle.shard_cost(x, d, dff) for x in L]
    whole = oracle.short_windows(L)
    # brute force: every contiguous partition whose cuts preserve the windows (reading s2)
    legal = [p for p in _all_partitions(B, R)
             if all(_windows_split_at(L, c) == whole for c in p[1:-1] if 0 < c < B)]
    best = min(max(sum(cost[p[r]:p[r + 1]]) for r in range(R)) for p in legal)
    plan = oracle.shard_plan(L, d, dff, R)
    assert plan in legal
    assert len(plan) == R + 1 and plan[0] == 0 and plan[-1] == B and plan == sorted(plan)
    assert max(sum(cost[plan[r]:plan[r + 1]]) for r in range(R)) == best
    # canonical: greedy-left at capacity `best` -> no rank could have ended at a later legal cut
    for r in range(R - 1):
        later = [q for q in legal if q[:r + 1] == plan[:r + 1] and q[r + 1] > plan[r + 1]
                 and sum(cost[plan[r]:q[r + 1]]) <= best]
        assert not later


def test_shard_cost_is_per_sequence_useful_flops():
    for L in (0, 1, 77, 512):
        assert oracle.shard_cost(L, 512, 2048) == oracle.useful_flops([L], 512, 2048)
