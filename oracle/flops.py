"""Analytic FLOP counts of the encoder layer (TEST INFRASTRUCTURE ONLY).

PAPER.md:133-142 (Fig. flop_ratios): relative FLOPs of the encoder layer with
and without padding, "computed analytically".  Readings c9 (padded = pad to
the batch maximum unless `pad_to` is given), c10 (FLOP = 2 MAC), c11 (only
matmul FLOPs on valid rows/columns are "useful").
"""
from __future__ import annotations

from typing import Optional, Sequence


def useful_flops(lengths: Sequence[int], d: int, d_ff: int) -> int:
    """2 * MACs of QKV, QK^T, AttnV, Proj, FF1, FF2 on the unpadded batch.

    MACs = T (3d^2 + d^2 + 2 d d_ff) + 2 d S2   with T = sum L, S2 = sum L^2.
    """
    T = sum(int(L) for L in lengths)
    S2 = sum(int(L) * int(L) for L in lengths)
    return 2 * (T * (4 * d * d + 2 * d * d_ff) + 2 * d * S2)


def padded_flops(lengths: Sequence[int], d: int, d_ff: int, pad_to: Optional[int] = None) -> int:
    """Same operators on the fully padded batch (every sequence padded to pad_to)."""
    Lp = max(int(L) for L in lengths) if pad_to is None else int(pad_to)
    return useful_flops([Lp] * len(lengths), d, d_ff)


def _loop_macs(lengths: Sequence[int], d: int, heads: int, d_ff: int) -> int:
    """Instrumented MAC count: literally walk the loop nests and count the inner bodies."""
    dh = d // heads
    macs = 0
    for L in lengths:
        L = int(L)
        for _i in range(L):           # token loop of the packed linear ops
            macs += 3 * d * d         # QKV: out 3d x in d
            macs += d * d             # Proj
            macs += d_ff * d          # FF1
            macs += d * d_ff          # FF2
        for _h in range(heads):
            for _i in range(L):
                for _j in range(L):
                    macs += dh        # QK^T  (reduction over d_h)
                    macs += dh        # AttnV (one MAC per output column per key)
    return macs


def useful_macs_bruteforce(lengths: Sequence[int], d: int, heads: int, d_ff: int) -> int:
    return _loop_macs(lengths, d, heads, d_ff)


def padded_macs_bruteforce(lengths: Sequence[int], d: int, heads: int, d_ff: int,
                           pad_to: Optional[int] = None) -> int:
    Lp = max(int(L) for L in lengths) if pad_to is None else int(pad_to)
    return _loop_macs([Lp] * len(lengths), d, heads, d_ff)


def qkt_macs(lengths: Sequence[int], heads: int, head_dim: int, pad_to: Optional[int] = None) -> int:
    """MACs of the QK^T operator alone: H * d_h * sum L^2 (ragged) or with every L -> pad_to."""
    if pad_to is not None:
        lengths = [int(pad_to)] * len(lengths)
    return heads * head_dim * sum(int(L) * int(L) for L in lengths)


def causal_attention_flops(lengths: Sequence[int], d: int) -> int:
    """Useful FLOPs of masked (causal) SDPA: QK^T and AttnV over the lower triangle incl. the diagonal,
    4 d * sum L (L + 1) / 2 ("a batch of lower triangular matrices")."""
    return 4 * d * sum(int(L) * (int(L) + 1) // 2 for L in lengths)
