"""Seeded synthetic inputs shared by the oracle (tests) and the CUDA path (bench).

This module holds NO arithmetic of the method (no offsets, no attention, no
LayerNorm): it only draws random numbers and rounds them to the storage
precision, so that the oracle (`oracle/`) and the product path
(`paper_2110_10221_b200/`) can consume identical inputs while sharing no code.

Recipe:

* Sequence lengths mimic the dataset statistics of PAPER.md:782-804
  (Table 3, "Datasets used in our evaluation": min / mean / max).  The real
  datasets are not available, so only min/mean/max are matched:
  ``L = clip(rint(min + (max-min) * Beta(a, b)), min, max)`` with
  ``a = kappa*m, b = kappa*(1-m), m = (mean-min)/(max-min), kappa = 4``,
  RNG ``numpy.random.Generator(PCG64(seed))``, default ``seed = 1000 + B``.
* Activations ``X ~ N(0, 1)``; Linear weights and biases ``~ U(+-1/sqrt(fan_in))``
  (nn.Linear init); LayerNorm ``gamma = 1 + 0.1 N(0,1)``, ``beta = 0.1 N(0,1)``.
  Data seed 0.  Matrices are rounded to bf16 once (round-to-nearest-even via
  torch's CPU cast); LayerNorm parameters are rounded to fp32.  The oracle
  consumes these rounded values exactly (they are exact in fp64).
"""
from __future__ import annotations

import dataclasses
from typing import Dict, Sequence

import numpy as np

# PAPER.md:790-799 (Table 3): min / mean / max sequence length per dataset.
DATASETS: Dict[str, tuple] = {
    "race": (80, 364, 512),
    "wiki512": (12, 371, 512),
    "squad": (39, 192, 384),
    "wiki128": (14, 117, 128),
    "mnli": (9, 43, 128),
    "xnli": (9, 70, 128),
    "mrpc": (21, 59, 102),
    "cola": (6, 13, 37),
}

KAPPA = 4.0


def dataset_lengths(name: str, batch: int, seed: int | None = None) -> np.ndarray:
    """Lengths drawn like dataset `name`, int64 [batch]."""
    mn, mean, mx = DATASETS[name]
    if seed is None:
        seed = 1000 + batch
    rng = np.random.Generator(np.random.PCG64(seed))
    m = (mean - mn) / (mx - mn)
    x = rng.beta(KAPPA * m, KAPPA * (1.0 - m), size=batch)
    return np.clip(np.rint(mn + (mx - mn) * x), mn, mx).astype(np.int64)


def uniform_lengths(batch: int, lo: int, hi: int, seed: int) -> np.ndarray:
    """U[lo, hi] integer lengths (padding sweep, config C5)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(lo, hi + 1, size=batch).astype(np.int64)


def skewed_lengths(batch: int, max_len: int, seed: int) -> np.ndarray:
    """One sequence of max_len, the rest log-normal(median 32, sigma 1) in [1, max_len] (C5)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    rest = np.clip(np.rint(np.exp(np.log(32.0) + rng.standard_normal(batch - 1))), 1, max_len)
    return np.concatenate([[max_len], rest]).astype(np.int64)


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round to the nearest bf16 (RNE) and return float64 holding the exact bf16 value."""
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def round_f32(a: np.ndarray) -> np.ndarray:
    return np.asarray(a, dtype=np.float32).astype(np.float64)


@dataclasses.dataclass
class EncoderWeights:
    """Weights of one post-LN encoder layer, nn.Linear convention W[out, in].

    All arrays are float64 holding exactly-representable bf16 (matrices, biases)
    or fp32 (LayerNorm) values.  Packing of W_qkv follows reading c5 of
    DESIGN.md: rows [0,d) = W_q, [d,2d) = W_k, [2d,3d) = W_v; head h uses rows
    [64h, 64h+64) within each block.
    """

    d_model: int
    heads: int
    d_ff: int
    w_qkv: np.ndarray
    b_qkv: np.ndarray
    w_o: np.ndarray
    b_o: np.ndarray
    ln1_g: np.ndarray
    ln1_b: np.ndarray
    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray
    ln2_g: np.ndarray
    ln2_b: np.ndarray


def encoder_weights(d_model: int, heads: int, d_ff: int, seed: int = 0) -> EncoderWeights:
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    d = d_model

    def lin(out_f, in_f):
        bound = 1.0 / np.sqrt(in_f)
        w = rng.uniform(-bound, bound, size=(out_f, in_f))
        b = rng.uniform(-bound, bound, size=(out_f,))
        return round_bf16(w), round_bf16(b)

    w_qkv, b_qkv = lin(3 * d, d)
    w_o, b_o = lin(d, d)
    w1, b1 = lin(d_ff, d)
    w2, b2 = lin(d, d_ff)
    ln1_g = round_f32(1.0 + 0.1 * rng.standard_normal(d))
    ln1_b = round_f32(0.1 * rng.standard_normal(d))
    ln2_g = round_f32(1.0 + 0.1 * rng.standard_normal(d))
    ln2_b = round_f32(0.1 * rng.standard_normal(d))
    return EncoderWeights(d, heads, d_ff, w_qkv, b_qkv, w_o, b_o, ln1_g, ln1_b, w1, b1, w2, b2, ln2_g, ln2_b)


def activations(total_tokens: int, cols: int, seed: int = 0) -> np.ndarray:
    """Packed activations X[T, cols] ~ N(0,1), bf16-exact float64."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return round_bf16(rng.standard_normal((total_tokens, cols)))


def normal(shape: Sequence[int], seed: int, scale: float = 1.0) -> np.ndarray:
    """Plain N(0, scale^2) float64 (not rounded)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return scale * rng.standard_normal(tuple(shape))


# The configurations of BASELINE.json "configs" (DESIGN.md section "Configs").
C1_LENGTHS = np.array([3, 7, 1, 5], dtype=np.int64)


def config(name: str):
    """Return (lengths, d_model, heads, d_ff) for a named configuration."""
    if name == "C1":
        return C1_LENGTHS.copy(), 16, 2, 32
    if name == "C2-mnli":
        return dataset_lengths("mnli", 32), 512, 8, 2048
    if name == "C2-mrpc":
        return dataset_lengths("mrpc", 32), 512, 8, 2048
    if name == "C3":
        return dataset_lengths("squad", 64), 512, 8, 2048
    if name == "C4-wiki512":
        return dataset_lengths("wiki512", 128), 512, 8, 2048
    if name == "C4-race":
        return dataset_lengths("race", 128), 512, 8, 2048
    # C5 padding-sensitivity sweep (BASELINE.json configs[4]): bs 32/64/128 x {all 512, U[1,512], skewed}
    if name.startswith("C5-"):
        _, kind, bs = name.split("-")
        B = int(bs)
        if kind == "equal":
            return np.full(B, 512, dtype=np.int64), 512, 8, 2048
        if kind == "uniform":
            return uniform_lengths(B, 1, 512, seed=2000 + B), 512, 8, 2048
        if kind == "skewed":
            return skewed_lengths(B, 512, seed=3000 + B), 512, 8, 2048
    # the other Table-3 datasets at bs 32/64/128: "<dataset>-<bs>"
    if "-" in name and name.split("-")[0] in DATASETS:
        ds, bs = name.split("-")
        return dataset_lengths(ds, int(bs)), 512, 8, 2048
    raise KeyError(name)


SWEEP_CONFIGS = ["C2-mnli", "C2-mrpc", "C3", "C4-wiki512", "C4-race"] + [
    f"C5-{k}-{b}" for k in ("equal", "uniform", "skewed") for b in (32, 64, 128)]
# the 24 cells of the paper's encoder-layer table (Table 4), synthetic lengths
TABLE4_CONFIGS = [f"{ds}-{b}" for ds in DATASETS for b in (32, 64, 128)]


def vgemm_dims(batch: int, seed: int, lo: int = 512, hi: int = 1408, step: int = 128) -> np.ndarray:
    """[batch, 3] (M_i, N_i, K_i), each an independent uniform multiple of `step` in [lo, hi]: the vgemm
    workload of PAPER.md:753-755 ("matrix dimensions are uniformly randomly chosen multiples of 128 in
    [512, 1408]")."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return (rng.integers(lo // step, hi // step + 1, size=(batch, 3)) * step).astype(np.int64)
