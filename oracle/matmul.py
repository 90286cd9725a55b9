"""vgemm and trmm (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

PAPER.md:738-851, Sec. "Matrix Multiplication":
  * vgemm -- "a batch of gemm operations, each with different dimensions", evaluated
    with "fully padded storage for all tensors" on "matrix dimensions ... uniformly
    randomly chosen multiples of 128 in [512, 1408]".  C_i = A_i B_i on the valid
    M_i x K_i / K_i x N_i blocks of the padded buffers; the padding of C is not part of the result.
  * trmm -- "multiply a square lower triangular matrix with a square dense matrix":
    C = tril(L) B, only the lower triangle of L (diagonal included) referenced (BLAS trmm semantics,
    reading f3-r1 in DESIGN.md); "the reduction loop is a vloop": row i reduces over
    k <= i.
Plain float64 NumPy; the library matmul is the step (no blocking).
"""
from __future__ import annotations

from typing import Sequence, Tuple

import numpy as np


def vgemm(a: np.ndarray, b: np.ndarray, dims: Sequence[Tuple[int, int, int]]) -> list:
    """[A_i[:M_i, :K_i] @ B_i[:K_i, :N_i] for each problem i] in float64 (a: [batch, M_max, K_max],
    b: [batch, K_max, N_max] padded buffers)."""
    out = []
    for i, (m, n, k) in enumerate(dims):
        out.append(np.asarray(a[i, :m, :k], np.float64) @ np.asarray(b[i, :k, :n], np.float64))
    return out


def trmm(l: np.ndarray, b: np.ndarray) -> np.ndarray:
    """tril(L) @ B in float64 (the strictly upper triangle of L is ignored)."""
    return np.tril(np.asarray(l, np.float64)) @ np.asarray(b, np.float64)


def vgemm_flops(dims: Sequence[Tuple[int, int, int]]) -> int:
    """Useful FLOPs (2 MAC) of the ragged batch: 2 sum_i M_i N_i K_i."""
    return 2 * sum(int(m) * int(n) * int(k) for m, n, k in dims)


def vgemm_padded_flops(dims: Sequence[Tuple[int, int, int]]) -> int:
    """FLOPs of the fully padded batched GEMM the paper compares against (every problem at the batch max)."""
    mm = max(int(d[0]) for d in dims)
    nn = max(int(d[1]) for d in dims)
    kk = max(int(d[2]) for d in dims)
    return 2 * len(dims) * mm * nn * kk


def trmm_flops(n: int, n_cols: int) -> int:
    """Useful FLOPs of tril(L) B: row i has i + 1 MACs per output column -> n (n + 1) / 2 * n_cols MACs."""
    return 2 * (n * (n + 1) // 2) * n_cols
