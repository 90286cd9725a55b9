"""Shared test helpers (no method arithmetic): error metric and GPU availability."""
import numpy as np
import pytest
import torch

HAVE_GPU = torch.cuda.is_available()
needs_gpu = pytest.mark.skipif(not HAVE_GPU, reason="no CUDA device")


def rel_err_rows(got, ref) -> float:
    """Reading c12 per row (reading c12b): max_i |g_i - o_i| / max(|o_i|, rms(row of o_i)), for
    attention outputs whose rows differ in scale by orders of magnitude -- a causal row i averages i + 1
    values, a row of a 4097-token sequence ~4097 -- where one tensor-wide rms would judge the large rows'
    bf16 rounding against the small rows' scale."""
    g = np.asarray(got, np.float64)
    o = np.asarray(ref, np.float64)
    if o.size == 0:
        return 0.0
    rms = np.sqrt(np.mean(o * o, axis=-1, keepdims=True))
    return float(np.max(np.abs(g - o) / np.maximum(np.abs(o), np.maximum(rms, 1e-300))))


def rel_err(got, ref) -> float:
    """Reading c12: max_i |g_i - o_i| / max(|o_i|, rms(o)) over one output tensor."""
    g = np.asarray(got, np.float64).ravel()
    o = np.asarray(ref, np.float64).ravel()
    if o.size == 0:
        return 0.0
    rms = float(np.sqrt(np.mean(o * o)))
    den = np.maximum(np.abs(o), rms if rms > 0 else 1.0)
    return float(np.max(np.abs(g - o) / den))


def to_np(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().double().numpy()


def bf16_cuda(a) -> torch.Tensor:
    return torch.as_tensor(np.asarray(a, np.float32)).to(torch.bfloat16).contiguous().cuda()


def f32_cuda(a) -> torch.Tensor:
    return torch.as_tensor(np.asarray(a, np.float32)).contiguous().cuda()


TOL_BF16 = 2e-2   # BASELINE.json north_star: bf16 tensor-core outputs
TOL_F32 = 1e-5    # BASELINE.json north_star: fp32 elementwise kernels
