"""Pins for oracle/layout.py: SPEC worked examples, brute-force enumeration, B.2 identities."""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_spec_row_offsets():
    for ex in GOLD["row_offsets"]:
        assert oracle.row_offsets(ex["lengths"]) == ex["expected"], ex["cite"]
    for ex in GOLD["total_size_2d"]:
        assert oracle.row_offsets(ex["lengths"])[-1] == ex["expected"], ex["cite"]


def test_spec_packed_offset():
    for ex in GOLD["packed_offset"]:
        ro = oracle.row_offsets(ex["lengths"])
        assert oracle.packed_offset(ro, *ex["index"], ex["d"]) == ex["expected"], ex["cite"]


def test_spec_attn_offsets():
    for ex in GOLD["attn_offsets"]:
        assert oracle.attn_offsets(ex["lengths"]) == ex["expected"], ex["cite"]
    for ex in GOLD["attn_offset"]:
        ao = oracle.attn_offsets(ex["lengths"])
        assert oracle.attn_offset(ao, ex["lengths"], ex["heads"], *ex["index"]) == ex["expected"], ex["cite"]
    for ex in GOLD["attn_total_size"]:
        assert oracle.attn_total_size(ex["lengths"], ex["heads"]) == ex["expected"], ex["cite"]


def test_spec_fusion_maps():
    for ex in GOLD["fusion_maps"]:
        f_fo, f_fi, base = oracle.fusion_maps(ex["lengths"])
        assert (f_fo, f_fi, base) == (ex["f_fo"], ex["f_fi"], ex["oif_base"]), ex["cite"]


def _enumerate_attention_layout(lengths, heads):
    """Walk X[b, i, h, j] in storage order (b, i, h, j) and record each position."""
    pos = {}
    k = 0
    for b, L in enumerate(lengths):
        for i in range(L):
            for h in range(heads):
                for j in range(L):
                    pos[(b, i, h, j)] = k
                    k += 1
    return pos, k


@pytest.mark.parametrize("lengths,heads", [([3, 7, 1, 5], 2), ([2, 3], 2), ([0, 4, 0, 1, 2], 3), ([5], 1)])
def test_attn_offset_is_enumeration_bijection(lengths, heads):
    pos, total = _enumerate_attention_layout(lengths, heads)
    ao = oracle.attn_offsets(lengths)
    assert oracle.attn_total_size(lengths, heads) == total
    got = {key: oracle.attn_offset(ao, lengths, heads, *key) for key in pos}
    assert got == pos
    assert sorted(got.values()) == list(range(total))


@pytest.mark.parametrize("lengths", [[3, 7, 1, 5], [0, 0, 2], [4]])
def test_packed_offset_is_enumeration_bijection(lengths):
    d = 3
    ro = oracle.row_offsets(lengths)
    k = 0
    for b, L in enumerate(lengths):
        for i in range(L):
            for c in range(d):
                assert oracle.packed_offset(ro, b, i, c, d) == k
                k += 1
    assert ro[-1] * d == k


def test_c1_tables_and_b2_identities():
    L = list(synth.C1_LENGTHS)
    f_fo, f_fi, base = oracle.fusion_maps(L)
    assert base == oracle.row_offsets(L)
    T = sum(L)
    for f in range(T):  # f_oif(f_fo(f), f_fi(f)) = f
        assert base[f_fo[f]] + f_fi[f] == f
    for o, Lo in enumerate(L):  # f_fo(f_oif(o,i)) = o, f_fi(f_oif(o,i)) = i
        for i in range(Lo):
            assert f_fo[base[o] + i] == o and f_fi[base[o] + i] == i


def test_descending_order_spec():
    for ex in GOLD["descending_order"]:
        # The tile rule with heads=1 and one tile per unit of work reproduces SortDescendingWork.
        lengths = [w * oracle.layout.Q_TILE for w in ex["work"]]
        seqs = []
        for b, _h, qt in oracle.tile_list(lengths, 1):
            if qt == 0:
                seqs.append(b)
        assert seqs == ex["expected"], ex["cite"]


@pytest.mark.parametrize("seed", range(5))
def test_tile_list_alternative_derivation(seed):
    rng = np.random.default_rng(seed)
    L = list(rng.integers(0, 700, size=int(rng.integers(1, 40))))
    H = int(rng.integers(1, 9))
    # Alternative derivation: stable sort sequences by descending tile count, then expand (h, qt).
    nq = [(x + 127) // 128 for x in L]
    order = sorted(range(len(L)), key=lambda b: -nq[b])  # Python sort is stable -> ties by b
    expect = [(b, h, qt) for b in order for h in range(H) for qt in range(nq[b])]
    assert oracle.tile_list(L, H) == expect
    assert oracle.n_tiles(L, H) == len(expect)


def test_validate_lengths():
    assert oracle.validate_lengths([3, 7, 1, 5], 16, 512) == oracle.STATUS_OK
    assert oracle.validate_lengths([3, 7, 1, 5], 17, 512) == oracle.STATUS_SUM_MISMATCH
    assert oracle.validate_lengths([3, -1, 1, 5], 8, 512) == oracle.STATUS_BAD_LENGTH
    assert oracle.validate_lengths([3, 600], 603, 512) == oracle.STATUS_BAD_LENGTH
    assert oracle.validate_lengths([3, 600], 5, 512) == oracle.STATUS_BAD_LENGTH | oracle.STATUS_SUM_MISMATCH
    assert oracle.validate_lengths([], 0, 512) == oracle.STATUS_OK


def test_synth_configs_match_survey():
    # The generator recipe of DESIGN.md reproduces the token counts quoted in SURVEY.md §8(d).
    for name, T, S2 in (("C4-wiki512", 47283, 18885603), ("C4-race", 46343, 17931033), ("C3", 12317, 2809789),
                        ("C2-mnli", 1465, 89879)):
        L, *_ = synth.config(name)
        assert int(L.sum()) == T and int((L ** 2).sum()) == S2


@pytest.mark.parametrize("seed", range(4))
def test_unit_list_alternative_derivation(seed):
    rng = np.random.default_rng(100 + seed)
    L = list(rng.integers(0, 700, size=int(rng.integers(1, 40))))
    H = int(rng.integers(1, 9))
    nq = [(x + 127) // 128 for x in L]
    order = sorted(range(len(L)), key=lambda b: -nq[b])
    expect = [(b, h, qp) for b in order for h in range(H) for qp in range((nq[b] + 1) // 2)]
    assert oracle.unit_list(L, H) == expect
    # every q-tile of the tile list is covered by exactly one unit (qt // 2 == qp)
    covered = sorted((b, h, qt) for b, h, qp in expect for qt in (2 * qp, 2 * qp + 1) if qt < nq[b])
    assert covered == sorted(oracle.tile_list(L, H))


def test_short_windows_examples():
    # tile 8 for readability: [3,4 | 2,2,2 | 9 | 5 | 0 ignored, 1] -> greedy windows in batch order
    L = [3, 4, 2, 2, 2, 9, 5, 0, 1]
    assert oracle.short_windows(L, tile=8) == [(0, 7, 2), (2, 6, 3), (6, 6, 2)]
    assert oracle.short_windows([], tile=8) == []
    assert oracle.short_windows([0, 0], tile=8) == []
    assert oracle.short_windows([8, 8], tile=8) == [(0, 8, 1), (1, 8, 1)]   # full tiles never merge
    assert oracle.short_windows([9, 1, 9], tile=8) == [(1, 1, 1)]


@pytest.mark.parametrize("seed", range(5))
def test_short_windows_invariants(seed):
    rng = np.random.default_rng(seed)
    L = [int(x) for x in rng.integers(0, 300, size=60)]
    ro = oracle.row_offsets(L)
    wins = oracle.short_windows(L)
    covered = []
    for b0, W, ns in wins:
        members = [b for b in range(b0, len(L)) if L[b] > 0][:ns]
        assert all(1 <= L[b] <= 128 for b in members)
        assert sum(L[b] for b in members) == W <= 128
        # contiguous in the packed token array: the members' rows are [ro[b0], ro[b0] + W)
        assert ro[members[-1]] + L[members[-1]] == ro[b0] + W
        covered += members
    assert covered == [b for b in range(len(L)) if 1 <= L[b] <= 128]  # every short sequence, once, in order
    # greedy maximality: the next short sequence after a window did not fit (or a long one intervened)
    for (b0, W, ns), nxt in zip(wins, wins[1:]):
        b1 = nxt[0]
        between = [b for b in range(b0, b1) if L[b] > 128]
        assert between or W + L[b1] > 128


def test_packed_lists_cover_the_same_rows():
    rng = np.random.default_rng(7)
    L = [int(x) for x in rng.integers(0, 400, size=40)]
    H = 3
    pt = oracle.packed_tile_list(L, H)
    plain = oracle.tile_list(L, H)
    long_items = [(b, h, qt) for b, h, qt, _p in pt if oracle.layout.n_q_tiles(L[b]) >= 2]
    assert long_items == [t for t in plain if oracle.layout.n_q_tiles(L[t[0]]) >= 2]
    n_win = len(oracle.short_windows(L))
    assert len(pt) == len(long_items) + H * n_win
    pu = oracle.packed_unit_list(L, H)
    assert len(pu) == len([u for u in oracle.unit_list(L, H) if oracle.layout.n_q_tiles(L[u[0]]) >= 2]) + H * n_win


# Hand-worked work lists (tile 8 for readability, 2 heads), derived on paper from reading f4-r1 (greedy
# windows in batch order, zero-length sequences transparent, a window with >= 2 members is `packed`) and
# the longest-first key (-q-tiles, b, h, qt) of reading c15: window order and
# packed bits are pinned item by item.
PACKED_CASES = [
    (
        [3, 4, 20, 2, 9, 1, 0, 5],  # q-tiles 1 1 3 1 2 1 0 1; windows {0,1} {3} {5,7}
        [(0, 7, 2), (3, 2, 1), (5, 6, 2)],
        [(2, 0, 0, 0), (2, 0, 1, 0), (2, 0, 2, 0), (2, 1, 0, 0), (2, 1, 1, 0), (2, 1, 2, 0),
         (4, 0, 0, 0), (4, 0, 1, 0), (4, 1, 0, 0), (4, 1, 1, 0),
         (0, 0, 0, 1), (0, 1, 0, 1), (3, 0, 0, 0), (3, 1, 0, 0), (5, 0, 0, 1), (5, 1, 0, 1)],
        [(2, 0, 0, 0), (2, 0, 1, 0), (2, 1, 0, 0), (2, 1, 1, 0), (4, 0, 0, 0), (4, 1, 0, 0),
         (0, 0, 0, 1), (0, 1, 0, 1), (3, 0, 0, 0), (3, 1, 0, 0), (5, 0, 0, 1), (5, 1, 0, 1)],
    ),
    (
        [8, 8, 1, 7, 0, 16, 2],  # q-tiles 1 1 1 1 0 2 1; full tiles never merge; windows {0} {1} {2,3} {6}
        [(0, 8, 1), (1, 8, 1), (2, 8, 2), (6, 2, 1)],
        [(5, 0, 0, 0), (5, 0, 1, 0), (5, 1, 0, 0), (5, 1, 1, 0),
         (0, 0, 0, 0), (0, 1, 0, 0), (1, 0, 0, 0), (1, 1, 0, 0), (2, 0, 0, 1), (2, 1, 0, 1), (6, 0, 0, 0), (6, 1, 0, 0)],
        [(5, 0, 0, 0), (5, 1, 0, 0),
         (0, 0, 0, 0), (0, 1, 0, 0), (1, 0, 0, 0), (1, 1, 0, 0), (2, 0, 0, 1), (2, 1, 0, 1), (6, 0, 0, 0), (6, 1, 0, 0)],
    ),
]


@pytest.mark.parametrize("L,wins,tiles,units", PACKED_CASES, ids=["mixed", "full-tiles"])
def test_packed_lists_hand_worked(L, wins, tiles, units):
    assert oracle.short_windows(L, tile=8) == wins
    assert oracle.packed_tile_list(L, 2, tile=8) == tiles
    assert oracle.packed_unit_list(L, 2, tile=8) == units
