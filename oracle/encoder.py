"""fp64 ragged encoder layer (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

The method (vloop fusion + ragged storage + minimal padding) computes exactly
the padded-and-masked dense encoder on the valid rows (PAPER.md:127-134,
929-932), so this oracle is that plain definition, evaluated one sequence at
a time in float64 with no padding at all.

Operator graph: PAPER.md:304-324 (Fig. fusion_graph) and the op list of
Table ap_op_times: QKV Proj (MM + bias) -> QK^T ->
Softmax -> AttnV -> Linear Proj MM + bias + ResidualAdd -> LayerNorm -> FF1 MM
+ bias + activation -> FF2 MM + bias + ResidualAdd -> LayerNorm.
Hyper-parameters: PAPER.md:908-912 (d_model 512, 8 heads x 64, FFN 2048).
Readings c1 (ReLU default, GELU-erf selectable), c2 (post-LN), c3 (eps 1e-5,
biased variance), c4 (scale 1/sqrt(d_h) applied to S), c5 (QKV packing
[W_q; W_k; W_v], head h = 64 contiguous columns), c6 (no dropout, no mask)
of DESIGN.md.
"""
from __future__ import annotations

import math
from typing import Optional, Sequence

import numpy as np
from scipy.special import erf

from .layout import attn_offset, attn_offsets, attn_total_size, row_offsets


def relu(x: np.ndarray) -> np.ndarray:
    return np.maximum(x, 0.0)


def gelu_erf(x: np.ndarray) -> np.ndarray:
    """GELU with the exact erf form, 0.5 x (1 + erf(x / sqrt 2)) (reading c1)."""
    return 0.5 * x * (1.0 + erf(x / math.sqrt(2.0)))


def linear(x: np.ndarray, w: np.ndarray, b: Optional[np.ndarray] = None,
           residual: Optional[np.ndarray] = None, act: Optional[str] = None) -> np.ndarray:
    """act(x W^T + b) + residual? -- "MM + Bias (+ Activation | + ResidualAdd)".

    PAPER.md:2255-2265 (Table ap_op_times rows QKV Proj, Linear Proj MM + Bias +
    ResidualAdd, FF1 MM + Bias + Activation, FF2 MM + Bias + ResidualAdd).
    The activation applies to the biased product; the residual is added after
    (the paper never combines both in one operator).  W uses nn.Linear [out, in].
    """
    y = np.asarray(x, np.float64) @ np.asarray(w, np.float64).T
    if b is not None:
        y = y + b
    if act == "relu":
        y = relu(y)
    elif act == "gelu":
        y = gelu_erf(y)
    elif act is not None:
        raise ValueError(act)
    if residual is not None:
        y = y + residual
    return y


def layernorm(y: np.ndarray, gamma: np.ndarray, beta: np.ndarray, eps: float = 1e-5) -> np.ndarray:
    """Row LayerNorm: gamma * (y - mu) / sqrt(var + eps) + beta, biased var (c3).

    PAPER.md:2262, 2266 ("LayerNorm" after the residual adds; c2 post-LN).
    """
    y = np.asarray(y, np.float64)
    mu = y.mean(axis=-1, keepdims=True)
    var = ((y - mu) ** 2).mean(axis=-1, keepdims=True)
    return (y - mu) / np.sqrt(var + eps) * gamma + beta


def softmax_row(s: np.ndarray) -> np.ndarray:
    """softmax over the last axis with max subtraction (Fig. ragged_softmax)."""
    s = np.asarray(s, np.float64)
    m = s.max(axis=-1, keepdims=True)
    e = np.exp(s - m)
    return e / e.sum(axis=-1, keepdims=True)


def attention_scores_ragged(qkv: np.ndarray, lengths: Sequence[int], heads: int) -> np.ndarray:
    """Scaled QK^T stored in CoRa's ragged attention layout X[b, i, h, j] (flat).

    PAPER.md:625-633 (X has cdims batch, head and vdims i, j of size s24(b)).
    """
    T, three_d = qkv.shape
    d = three_d // 3
    dh = d // heads
    row_off = row_offsets(lengths)
    a_off = attn_offsets(lengths)
    out = np.zeros(attn_total_size(lengths, heads), np.float64)
    for b, L in enumerate(lengths):
        L = int(L)
        r0 = row_off[b]
        for h in range(heads):
            q = qkv[r0:r0 + L, h * dh:(h + 1) * dh]
            k = qkv[r0:r0 + L, d + h * dh:d + (h + 1) * dh]
            s = (q @ k.T) * (1.0 / math.sqrt(dh))
            for i in range(L):
                o = attn_offset(a_off, lengths, heads, b, i, h, 0)
                out[o:o + L] = s[i]
    return out


def ragged_softmax(x_flat: np.ndarray, lengths: Sequence[int], heads: int) -> np.ndarray:
    """Softmax of every row X[b, i, h, 0:L_b] of the ragged attention matrix.

    PAPER.md:2255-2258 ("ChangePad + Softmax + ChangePad") on the layout of
    PAPER.md:625-633; rows are addressed with the lowered offsets of B.1.
    """
    a_off = attn_offsets(lengths)
    out = np.zeros_like(np.asarray(x_flat, np.float64))
    for b, L in enumerate(lengths):
        L = int(L)
        for i in range(L):
            for h in range(heads):
                o = attn_offset(a_off, lengths, heads, b, i, h, 0)
                out[o:o + L] = softmax_row(x_flat[o:o + L])
    return out


def ragged_attention(qkv: np.ndarray, lengths: Sequence[int], heads: int, causal: bool = False) -> np.ndarray:
    """O[T, d] = concat_h softmax(Q_h K_h^T / sqrt(d_h)) V_h per sequence.

    PAPER.md:296-300 (SDPA sub-module), 2256-2259 (QK^T, Softmax, AttnV);
    only j < L_b exist (no padded keys, no mask within a sequence: encoder).
    causal=True: the masked MHA of the decoder (App. D.3
    1752-1806): "the upper half of the attention matrix is masked", i.e. query
    i attends to keys j <= i of its own sequence only (lower-triangular S).
    """
    T, three_d = qkv.shape
    d = three_d // 3
    dh = d // heads
    row_off = row_offsets(lengths)
    out = np.zeros((T, d), np.float64)
    for b, L in enumerate(lengths):
        L = int(L)
        if L == 0:
            continue
        r0 = row_off[b]
        for h in range(heads):
            q = qkv[r0:r0 + L, h * dh:(h + 1) * dh]
            k = qkv[r0:r0 + L, d + h * dh:d + (h + 1) * dh]
            v = qkv[r0:r0 + L, 2 * d + h * dh:2 * d + (h + 1) * dh]
            sc = (q @ k.T) * (1.0 / math.sqrt(dh))
            if causal:
                sc = np.where(np.tril(np.ones((L, L), dtype=bool)), sc, -np.inf)
            p = softmax_row(sc)
            out[r0:r0 + L, h * dh:(h + 1) * dh] = p @ v
    return out


def ragged_attention_rows(qkv: np.ndarray, lengths: Sequence[int], heads: int, rows: Sequence[int],
                          causal: bool = False) -> np.ndarray:
    """The rows `rows` (packed token indices) of ragged_attention, one at a time: for token t of sequence b
    (position i), O[t, h] = softmax_j(q_t . k_j / sqrt(d_h)) v_j over the keys j < L_b of its own sequence
    (j <= i when causal) -- the same definition, for sequences too long to
    form their L x L score matrices (max_len 16383).  Returns [len(rows), d]."""
    T, three_d = qkv.shape
    d = three_d // 3
    dh = d // heads
    row_off = row_offsets(lengths)
    out = np.zeros((len(rows), d), np.float64)
    for n, t in enumerate(rows):
        b = int(np.searchsorted(row_off, t, side="right")) - 1
        while int(lengths[b]) == 0:  # zero-length sequences share their row offset with the next one
            b += 1
        r0, L = row_off[b], int(lengths[b])
        i = t - r0
        nk = i + 1 if causal else L
        for h in range(heads):
            q = qkv[t, h * dh:(h + 1) * dh]
            k = qkv[r0:r0 + nk, d + h * dh:d + (h + 1) * dh]
            v = qkv[r0:r0 + nk, 2 * d + h * dh:2 * d + (h + 1) * dh]
            p = softmax_row((k @ q) * (1.0 / math.sqrt(dh)))
            out[n, h * dh:(h + 1) * dh] = p @ v
    return out


def encoder_layer(x: np.ndarray, lengths: Sequence[int], w, eps: float = 1e-5, act: str = "relu",
                  return_intermediates: bool = False):
    """Forward pass of one post-LN encoder layer over a ragged batch, fp64.

    x: packed tokens [T, d] (T = sum L_b, sequence b at rows row_off[b]..).
    w: synth.EncoderWeights (or any object with the same attributes).
    Steps 1-9 of DESIGN.md "Oracle", one sequence at a time.
    """
    x = np.asarray(x, np.float64)
    T, d = x.shape
    row_off = row_offsets(lengths)
    assert row_off[-1] == T
    inter = {k: np.zeros((T, n)) for k, n in
             (("qkv", 3 * d), ("attn", d), ("y1", d), ("h1", d), ("f", w.d_ff), ("y2", d), ("out", d))}
    for b, L in enumerate(lengths):
        L = int(L)
        if L == 0:
            continue
        rows = slice(row_off[b], row_off[b] + L)
        xs = x[rows]
        qkv = linear(xs, w.w_qkv, w.b_qkv)                                   # 1
        attn = ragged_attention(qkv, [L], w.heads)                            # 2-4
        y1 = linear(attn, w.w_o, w.b_o, residual=xs)                          # 5
        h1 = layernorm(y1, w.ln1_g, w.ln1_b, eps)                             # 6
        f = linear(h1, w.w1, w.b1, act=act)                                   # 7
        y2 = linear(f, w.w2, w.b2, residual=h1)                               # 8
        out = layernorm(y2, w.ln2_g, w.ln2_b, eps)                            # 9
        for k, v in (("qkv", qkv), ("attn", attn), ("y1", y1), ("h1", h1), ("f", f), ("y2", y2), ("out", out)):
            inter[k][rows] = v
    if return_intermediates:
        return inter
    return inter["out"]
