"""Pins for oracle/encoder.py against independent implementations (torch fp64) and invariants."""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
torch.set_default_dtype(torch.float64)


def _t(a):
    return torch.from_numpy(np.asarray(a, np.float64))


def test_spec_softmax_row():
    for ex in GOLD["softmax_row"]:
        assert np.allclose(oracle.softmax_row(np.array(ex["row"])), ex["expected"], atol=0, rtol=0), ex["cite"]


def test_linear_vs_python_loops():
    rng = np.random.default_rng(1)
    x, w, b, r = rng.standard_normal((5, 4)), rng.standard_normal((3, 4)), rng.standard_normal(3), rng.standard_normal((5, 3))
    for act in (None, "relu", "gelu"):
        got = oracle.linear(x, w, b, residual=r, act=act)
        for i in range(5):
            for n in range(3):
                acc = b[n]
                for k in range(4):
                    acc += x[i, k] * w[n, k]
                if act == "relu":
                    acc = max(acc, 0.0)
                elif act == "gelu":
                    acc = 0.5 * acc * (1.0 + math.erf(acc / math.sqrt(2.0)))
                assert abs(got[i, n] - (acc + r[i, n])) < 1e-13


def test_layernorm_vs_torch_and_moments():
    rng = np.random.default_rng(2)
    y = rng.standard_normal((7, 512)) * 3 + 1
    g, b = rng.standard_normal(512), rng.standard_normal(512)
    ref = torch.nn.functional.layer_norm(_t(y), (512,), _t(g), _t(b), eps=1e-5).numpy()
    assert np.abs(oracle.layernorm(y, g, b, 1e-5) - ref).max() < 1e-12
    # gamma = 1, beta = 0: row mean 0, row (biased) variance sigma^2/(sigma^2+eps)
    out = oracle.layernorm(y, np.ones(512), np.zeros(512), 1e-5)
    var = y.var(axis=1)
    assert np.abs(out.mean(axis=1)).max() < 1e-13
    assert np.abs(out.var(axis=1) - var / (var + 1e-5)).max() < 1e-12


def _qkv(lengths, d, seed=3):
    return synth.normal((sum(lengths), 3 * d), seed)


def test_attention_b1_is_textbook_sdpa():
    L, H, d = 37, 4, 32
    qkv = _qkv([L], d)
    got = oracle.ragged_attention(qkv, [L], H)
    q, k, v = (_t(qkv[:, i * d:(i + 1) * d]).reshape(L, H, d // H).transpose(0, 1) for i in range(3))
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v).transpose(0, 1).reshape(L, d).numpy()
    assert np.abs(got - ref).max() < 1e-13


def test_attention_vs_padded_masked_dense():
    lengths, H, d = [3, 7, 1, 5, 0, 2], 2, 16
    qkv = _qkv(lengths, d, seed=4)
    got = oracle.ragged_attention(qkv, lengths, H)
    B, Lp, dh = len(lengths), max(lengths), d // H
    ro = oracle.row_offsets(lengths)
    pad = torch.zeros(B, Lp, 3 * d)
    mask = torch.ones(B, Lp, dtype=torch.bool)  # True = valid key
    for b, L in enumerate(lengths):
        pad[b, :L] = _t(qkv[ro[b]:ro[b] + L])
        mask[b, L:] = False
    q, k, v = (pad[..., i * d:(i + 1) * d].reshape(B, Lp, H, dh).transpose(1, 2) for i in range(3))
    attn_mask = mask[:, None, None, :].expand(B, H, Lp, Lp).clone()
    attn_mask[:, :, :, 0] |= ~mask[:, None, :].expand(B, H, Lp)  # keep fully-padded query rows finite
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, attn_mask=attn_mask).transpose(1, 2).reshape(B, Lp, d)
    for b, L in enumerate(lengths):
        if L:
            assert np.abs(got[ro[b]:ro[b] + L] - ref[b, :L].numpy()).max() < 1e-13


def test_attention_invariants():
    d, H = 16, 2
    # L = 1: softmax of one score is exactly 1, so O = V.
    qkv = _qkv([1], d, seed=5)
    assert np.array_equal(oracle.ragged_attention(qkv, [1], H), qkv[:, 2 * d:])
    # Identical keys: every row of P is uniform, so O = mean of V.
    qkv = _qkv([6], d, seed=6)
    qkv[:, d:2 * d] = qkv[0, d:2 * d]
    out = oracle.ragged_attention(qkv, [6], H)
    assert np.abs(out - qkv[:, 2 * d:].mean(axis=0)).max() < 1e-14
    # A sequence's output does not depend on its neighbours (padding / neighbours never leak).
    lengths = [4, 5, 3]
    qkv = _qkv(lengths, d, seed=7)
    a = oracle.ragged_attention(qkv, lengths, H)
    qkv2 = qkv.copy()
    qkv2[4:9] += 10.0
    b = oracle.ragged_attention(qkv2, lengths, H)
    assert np.array_equal(a[:4], b[:4]) and np.array_equal(a[9:], b[9:])


def test_ragged_softmax_rows_and_layout():
    lengths, H, d = [3, 7, 1, 5], 2, 16
    qkv = _qkv(lengths, d, seed=8)
    x = oracle.attention_scores_ragged(qkv, lengths, H)
    p = oracle.ragged_softmax(x, lengths, H)
    ao = oracle.attn_offsets(lengths)
    for b, L in enumerate(lengths):
        for i in range(L):
            for h in range(H):
                o = oracle.attn_offset(ao, lengths, H, b, i, h, 0)
                assert abs(p[o:o + L].sum() - 1.0) < 1e-15
                ref = torch.softmax(_t(x[o:o + L]), 0).numpy()
                assert np.abs(p[o:o + L] - ref).max() < 1e-15
    # shift invariance of every row
    assert np.abs(oracle.ragged_softmax(x + 3.0, lengths, H) - p).max() < 1e-14
    # softmax(scores) @ V reproduces the fused attention
    out = oracle.ragged_attention(qkv, lengths, H)
    ro = oracle.row_offsets(lengths)
    dh = d // H
    for b, L in enumerate(lengths):
        for h in range(H):
            P = np.stack([p[oracle.attn_offset(ao, lengths, H, b, i, h, 0):][:L] for i in range(L)])
            V = qkv[ro[b]:ro[b] + L, 2 * d + h * dh:2 * d + (h + 1) * dh]
            assert np.abs(P @ V - out[ro[b]:ro[b] + L, h * dh:(h + 1) * dh]).max() < 1e-13


def _torch_layer(w, act):
    layer = torch.nn.TransformerEncoderLayer(w.d_model, w.heads, w.d_ff, dropout=0.0, activation=act,
                                             batch_first=True, norm_first=False, dtype=torch.float64)
    with torch.no_grad():
        layer.self_attn.in_proj_weight.copy_(_t(w.w_qkv))
        layer.self_attn.in_proj_bias.copy_(_t(w.b_qkv))
        layer.self_attn.out_proj.weight.copy_(_t(w.w_o))
        layer.self_attn.out_proj.bias.copy_(_t(w.b_o))
        layer.linear1.weight.copy_(_t(w.w1))
        layer.linear1.bias.copy_(_t(w.b1))
        layer.linear2.weight.copy_(_t(w.w2))
        layer.linear2.bias.copy_(_t(w.b2))
        layer.norm1.weight.copy_(_t(w.ln1_g))
        layer.norm1.bias.copy_(_t(w.ln1_b))
        layer.norm2.weight.copy_(_t(w.ln2_g))
        layer.norm2.bias.copy_(_t(w.ln2_b))
    return layer.train(False)


@pytest.mark.parametrize("act", ["relu", "gelu"])
def test_encoder_layer_vs_torch_c1(act):
    lengths, d, H, dff = synth.config("C1")
    w = synth.encoder_weights(d, H, dff)
    x = synth.activations(int(lengths.sum()), d)
    got = oracle.encoder_layer(x, lengths, w, act=act)
    layer = _torch_layer(w, act)
    ro = oracle.row_offsets(lengths)
    # per sequence
    for b, L in enumerate(lengths):
        ref = layer(_t(x[ro[b]:ro[b] + L])[None]).detach()[0].numpy()
        assert np.abs(got[ro[b]:ro[b] + L] - ref).max() < 1e-12
    # padded batch with src_key_padding_mask (the padded-and-masked dense computation)
    B, Lp = len(lengths), int(lengths.max())
    pad = torch.zeros(B, Lp, d)
    mask = torch.zeros(B, Lp, dtype=torch.bool)  # True = padding
    for b, L in enumerate(lengths):
        pad[b, :L] = _t(x[ro[b]:ro[b] + L])
        mask[b, L:] = True
    ref = layer(pad, src_key_padding_mask=mask).detach().numpy()
    for b, L in enumerate(lengths):
        assert np.abs(got[ro[b]:ro[b] + L] - ref[b, :L]).max() < 1e-12


def test_encoder_layer_vs_torch_full_width():
    # d_model 512, 8 heads, FFN 2048 on a short ragged batch.
    lengths = np.array([9, 1, 30, 17])
    w = synth.encoder_weights(512, 8, 2048, seed=1)
    x = synth.activations(int(lengths.sum()), 512, seed=1)
    got = oracle.encoder_layer(x, lengths, w)
    layer = _torch_layer(w, "relu")
    ro = oracle.row_offsets(lengths)
    for b, L in enumerate(lengths):
        ref = layer(_t(x[ro[b]:ro[b] + L])[None]).detach()[0].numpy()
        assert np.abs(got[ro[b]:ro[b] + L] - ref).max() < 1e-11


def test_encoder_layer_zero_length_sequences():
    lengths = np.array([0, 3, 0, 2, 0])
    w = synth.encoder_weights(16, 2, 32)
    x = synth.activations(5, 16)
    got = oracle.encoder_layer(x, lengths, w)
    alone = np.concatenate([oracle.encoder_layer(x[:3], [3], w), oracle.encoder_layer(x[3:], [2], w)])
    assert np.array_equal(got, alone)


def test_causal_attention_b1_is_textbook_causal_sdpa():
    L, H, d = 29, 2, 16
    qkv = _qkv([L], d, seed=9)
    got = oracle.ragged_attention(qkv, [L], H, causal=True)
    q, k, v = (_t(qkv[:, i * d:(i + 1) * d]).reshape(L, H, d // H).transpose(0, 1) for i in range(3))
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True).transpose(0, 1).reshape(L, d).numpy()
    assert np.abs(got - ref).max() < 1e-13


def test_causal_attention_invariants():
    lengths, H, d = [5, 1, 7], 2, 16
    qkv = _qkv(lengths, d, seed=10)
    out = oracle.ragged_attention(qkv, lengths, H, causal=True)
    ro = oracle.row_offsets(lengths)
    # the first query of every sequence sees only its own key: O = V exactly
    for b in range(len(lengths)):
        assert np.array_equal(out[ro[b]], qkv[ro[b], 2 * d:])
    # the last query of a sequence sees every key: identical to the unmasked row
    full = oracle.ragged_attention(qkv, lengths, H)
    for b, L in enumerate(lengths):
        assert np.abs(out[ro[b] + L - 1] - full[ro[b] + L - 1]).max() < 1e-14
    # row i does not depend on later keys of its sequence
    qkv2 = qkv.copy()
    qkv2[ro[2] + 4:ro[2] + 7, d:] += 5.0
    out2 = oracle.ragged_attention(qkv2, lengths, H, causal=True)
    assert np.array_equal(out[:ro[2] + 4], out2[:ro[2] + 4])
    # FLOP count of the lower triangle
    assert oracle.causal_attention_flops([3], 8) == 4 * 8 * 6


@pytest.mark.parametrize("causal", [False, True])
def test_attention_rows_vs_torch_sdpa(causal):
    """ragged_attention_rows (the row-at-a-time form for sequences too long for an L x L score matrix) against
    torch SDPA fp64 per sequence (is_causal for the masked variant), on sampled rows of a batch with zero-length
    sequences, a 1-token sequence and a sequence of 700 tokens (6 q-tiles)."""
    lengths, H, d = [0, 700, 1, 0, 130, 5], 4, 64
    qkv = _qkv(lengths, d, seed=11)
    ro = oracle.row_offsets(lengths)
    rows = [0, 1, 127, 128, 511, 699, 700, 701, 790, 830, 831, 835]
    got = oracle.ragged_attention_rows(qkv, lengths, H, rows, causal=causal)
    for n, t in enumerate(rows):
        b = max(i for i in range(len(lengths)) if ro[i] <= t and lengths[i] > 0)
        L, r0 = lengths[b], ro[b]
        seq = qkv[r0:r0 + L]
        q, k, v = (_t(seq[:, i * d:(i + 1) * d]).reshape(L, H, d // H).transpose(0, 1) for i in range(3))
        ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=causal).transpose(0, 1).reshape(L, d)
        assert np.abs(got[n] - ref[t - r0].numpy()).max() < 1e-13, (t, causal)
