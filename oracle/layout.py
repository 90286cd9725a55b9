"""Offset tables of CoRa's ragged storage (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Paper passages followed:
* PAPER.md:584-604 (§5.1 "Loop and Tensor Dimension Fusion"): the fused loop
  bound F = sum_o s(o) and the mapping between fused and unfused iteration
  variables, computed in the prelude.
* PAPER.md:1583-1616 (App. B.1): the auxiliary function A_d, e.g. for the
  attention matrix X, A_1[i] = sum_j s24(j)*s24(j); Algorithm 1
   lowers an access to a flat offset.  Reading c7: we use
  EXCLUSIVE prefixes (A[0] = 0), as SPEC.md:169-170 does.
* PAPER.md:1618-1642 (App. B.2): fusion maps f_fo, f_fi, f_oif and their
  identities f_oif(f_fo(f), f_fi(f)) = f, ...
* PAPER.md:1736-1750 (App. D.2 "Load Balancing"): sequences are sorted in
  descending order of length "so that thread blocks with the most amount of
  work are scheduled first".  Reading c15: the attention work list is every
  (b, h, qt) with qt < ceil(L_b/128), ordered by the key
  (-ceil(L_b/128), b, h, qt) -- ties go to the lower id.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

STATUS_OK = 0
STATUS_BAD_LENGTH = 1  # some L_b < 0 or L_b > max_len
STATUS_SUM_MISMATCH = 2  # sum_b L_b != total_tokens

Q_TILE = 128  # rows of one attention work tile (the sm_100a UMMA M)


def row_offsets(lengths: Sequence[int]) -> List[int]:
    """A_1 of the packed [b, i, c] layout: row_off[b] = sum_{j<b} L_j, len B+1.

    PAPER.md:598-604 (fused bound F = sum_o s(o)) and PAPER.md:1583-1593
    (A_d as a CSR-like row_index array), exclusive convention (reading c7).
    """
    out = [0]
    for L in lengths:
        out.append(out[-1] + int(L))
    return out


def attn_offsets(lengths: Sequence[int]) -> List[int]:
    """A_1 of the attention matrix X[b, i, h, j]: attn_off[b] = sum_{j<b} L_j^2.

    PAPER.md:1589-1593: "A_1[i] = sum_{j=1}^{i} s24(j)*s24(j)" (exclusive, c7).
    """
    out = [0]
    for L in lengths:
        out.append(out[-1] + int(L) * int(L))
    return out


def fusion_maps(lengths: Sequence[int]) -> Tuple[List[int], List[int], List[int]]:
    """(f_fo, f_fi, oif_base) of PAPER.md:1622-1642 (App. B.2).

    f_fo[f] = o and f_fi[f] = i for the fused index f of the loop nest
    `for o: for i < s(o)` (Fig. fusion); f_oif(o, i) =
    oif_base[o] + i.  Built by literally running the unfused loop nest.
    """
    f_fo: List[int] = []
    f_fi: List[int] = []
    oif_base: List[int] = []
    f = 0
    for o, L in enumerate(lengths):
        oif_base.append(f)
        for i in range(int(L)):
            f_fo.append(o)
            f_fi.append(i)
            f += 1
    oif_base.append(f)
    return f_fo, f_fi, oif_base


def packed_offset(row_off: Sequence[int], b: int, i: int, c: int, d: int) -> int:
    """Flat offset of element (b, i, c) of a [batch, len_b (vdim), d (cdim)] tensor.

    Algorithm 1 for the dgraph {1->2}: D = A_1(b)*d + i*d + c.
    """
    return row_off[b] * d + i * d + c


def attn_offset(attn_off: Sequence[int], lengths: Sequence[int], heads: int, b: int, i: int, h: int, j: int) -> int:
    """Flat offset of X[b, i, h, j] (PAPER.md:625-633 layout, B.1 lowering).

    Dims (batch, seq_i, head, seq_j) with s2 = s4 = s24(b);
    A_1 covers dims 2..4 (O*_G(1) = {2, 4}, times the cdim 3), so
    offset = H*A_1(b) + i*H*L_b + h*L_b + j   (reading c8).
    """
    L = int(lengths[b])
    return heads * attn_off[b] + i * heads * L + h * L + j


def attn_total_size(lengths: Sequence[int], heads: int) -> int:
    return heads * sum(int(L) * int(L) for L in lengths)


def n_q_tiles(L: int, tile: int = Q_TILE) -> int:
    return (int(L) + tile - 1) // tile


def tile_list(lengths: Sequence[int], heads: int, tile: int = Q_TILE) -> List[Tuple[int, int, int]]:
    """Longest-first attention work list (reading c15).

    Plain definition: enumerate every (b, h, qt), then sort by the key.
    """
    items = []
    for b, L in enumerate(lengths):
        for h in range(heads):
            for qt in range(n_q_tiles(L, tile)):
                items.append((b, h, qt))
    items.sort(key=lambda t: (-n_q_tiles(lengths[t[0]], tile), t[0], t[1], t[2]))
    return items


def unit_list(lengths: Sequence[int], heads: int, tile: int = Q_TILE) -> List[Tuple[int, int, int]]:
    """Attention work units: pairs of consecutive q-tiles of one (sequence, head) that share their
    K/V tiles, (b, h, qp) for qp < ceil(ceil(L_b/128)/2), same longest-first key as tile_list
    (reading c15).  Plain definition: enumerate, then sort."""
    items = []
    for b, L in enumerate(lengths):
        npairs = (n_q_tiles(L, tile) + 1) // 2
        for h in range(heads):
            for qp in range(npairs):
                items.append((b, h, qp))
    items.sort(key=lambda t: (-n_q_tiles(lengths[t[0]], tile), t[0], t[1], t[2]))
    return items


def short_windows(lengths: Sequence[int], tile: int = Q_TILE) -> List[Tuple[int, int, int]]:
    """Windows of consecutive short sequences (SURVEY f-4; reading f4-r1 of DESIGN.md).

    Sequences with 1 <= L_b <= tile occupy one q-tile each, mostly masked lanes when short (the partial
    padding whose cost grows for short sequences).  Consecutive short sequences are
    contiguous in the packed token array, so a 128-row window of them is one attention tile whose score
    block is block-diagonal.  Greedy in batch order: a short sequence joins the open window if the
    window's token count stays <= tile, else it opens a new window; a sequence longer than the tile
    closes the open window; zero-length sequences are transparent.
    Returns [(b_first, W tokens, n_seq)] in batch order."""
    wins = []
    cur = None  # [b_first, W, n_seq]
    for b, L in enumerate(lengths):
        L = int(L)
        if L == 0:
            continue
        if L > tile:
            if cur is not None:
                wins.append(tuple(cur))
                cur = None
            continue
        if cur is not None and cur[1] + L <= tile:
            cur[1] += L
            cur[2] += 1
        else:
            if cur is not None:
                wins.append(tuple(cur))
            cur = [b, L, 1]
    if cur is not None:
        wins.append(tuple(cur))
    return wins


def packed_tile_list(lengths: Sequence[int], heads: int, tile: int = Q_TILE) -> List[Tuple[int, int, int, int]]:
    """The device work list with short-sequence packing: (b, h, qt, packed).

    Sequences with more than one q-tile contribute (b, h, qt, 0) as in tile_list; the short sequences
    contribute one item per (window, head) instead, (b_first, h, 0, n_seq >= 2).  Longest-first key
    (-q-tiles, b, h, qt) as in tile_list (reading c15), a window keyed by its first
    sequence.  Plain definition: enumerate, then sort."""
    items = []
    for b, L in enumerate(lengths):
        if n_q_tiles(L, tile) >= 2:
            for h in range(heads):
                for qt in range(n_q_tiles(L, tile)):
                    items.append((n_q_tiles(L, tile), b, h, qt, 0))
    for b0, _w, ns in short_windows(lengths, tile):
        for h in range(heads):
            items.append((1, b0, h, 0, 1 if ns >= 2 else 0))
    items.sort(key=lambda t: (-t[0], t[1], t[2], t[3]))
    return [t[1:] for t in items]


def packed_unit_list(lengths: Sequence[int], heads: int, tile: int = Q_TILE) -> List[Tuple[int, int, int, int]]:
    """unit_list with the same short-sequence windows: (b, h, qp, packed)."""
    items = []
    for b, L in enumerate(lengths):
        nq = n_q_tiles(L, tile)
        if nq >= 2:
            for h in range(heads):
                for qp in range((nq + 1) // 2):
                    items.append((nq, b, h, qp, 0))
    for b0, _w, ns in short_windows(lengths, tile):
        for h in range(heads):
            items.append((1, b0, h, 0, 1 if ns >= 2 else 0))
    items.sort(key=lambda t: (-t[0], t[1], t[2], t[3]))
    return [t[1:] for t in items]


def n_tiles(lengths: Sequence[int], heads: int, tile: int = Q_TILE) -> int:
    return heads * sum(n_q_tiles(L, tile) for L in lengths)


def validate_lengths(lengths: Sequence[int], total_tokens: int, max_len: int) -> int:
    """Status word of the layout builder (SPEC.md:619-623 SizeMismatch, 643 exit codes)."""
    status = STATUS_OK
    if any(int(L) < 0 or int(L) > max_len for L in lengths):
        status |= STATUS_BAD_LENGTH
    if sum(int(L) for L in lengths) != total_tokens:
        status |= STATUS_SUM_MISMATCH
    return status
