"""GPU parity of vgemm / trmm (SURVEY f-3) through the C ABI against the fp64 oracle."""
import numpy as np
import pytest
import torch

import oracle
import synth
from util import TOL_BF16, bf16_cuda, rel_err, to_np

pytestmark = pytest.mark.gpu


def P():
    import paper_2110_10221_b200 as P
    return P


VGEMM_CASES = [
    [(128, 256, 64)],                                    # one tile
    [(512, 640, 512), (1408, 512, 1408), (640, 1408, 768)],  # the paper's range, ragged N tiles
    [(100, 72, 128), (1, 8, 64), (0, 16, 64), (257, 264, 192), (33, 0, 64)],  # M/N tails, empty problems
    [(300, 200, 200)],                                   # K tail == K_max (TMA zero-fill)
    [(64, 64, 0), (128, 256, 64), (200, 100, 0)],        # K_i == 0: C_i = 0 (no stale accumulator)
]


@pytest.mark.parametrize("dims", VGEMM_CASES, ids=lambda d: f"B{len(d)}")
def test_vgemm_parity_and_untouched_padding(dims):
    batch = len(dims)
    mm = max(d[0] for d in dims)
    nn = max(8, -(-max(d[1] for d in dims) // 8) * 8)
    kk = max(8, -(-max(d[2] for d in dims) // 8) * 8)
    a = synth.round_bf16(synth.normal((batch, mm, kk), 11))
    b = synth.round_bf16(synth.normal((batch, kk, nn), 12) / np.sqrt(kk))
    sentinel = torch.full((batch, mm, nn), 7.0, dtype=torch.bfloat16, device="cuda")
    c = to_np(P().vgemm(bf16_cuda(a), bf16_cuda(b), dims, out=sentinel))
    ref = oracle.vgemm(a, b, dims)
    for i, (m, n, k) in enumerate(dims):
        assert rel_err(c[i, :m, :n], ref[i]) <= TOL_BF16
        pad = np.ones((mm, nn), bool)
        pad[:m, :n] = False
        assert np.all(c[i][pad] == 7.0)  # the padding of C is never written


def test_vgemm_paper_workload_sample():
    d = synth.vgemm_dims(16, seed=3)
    dims = [tuple(map(int, r)) for r in d]
    mm, nn, kk = (int(d[:, j].max()) for j in range(3))
    a = synth.round_bf16(synth.normal((16, mm, kk), 13))
    b = synth.round_bf16(synth.normal((16, kk, nn), 14) / np.sqrt(kk))
    c = to_np(P().vgemm(bf16_cuda(a), bf16_cuda(b), dims))
    ref = oracle.vgemm(a, b, dims)
    for i, (m, n, k) in enumerate(dims):
        assert rel_err(c[i, :m, :n], ref[i]) <= TOL_BF16


def test_vgemm_in_a_cuda_graph():
    """The plan lives in pinned host memory, so the call (plan copy + kernel) is stream-capturable; a replay
    recomputes C after the inputs change."""
    dims = [(300, 200, 256), (128, 264, 64), (0, 8, 64), (257, 64, 128)]
    mm, nn, kk = 300, 264, 256
    a = synth.round_bf16(synth.normal((4, mm, kk), 31))
    b = synth.round_bf16(synth.normal((4, kk, nn), 32) / np.sqrt(kk))
    ta, tb = bf16_cuda(a), bf16_cuda(b)
    c = torch.zeros(4, mm, nn, dtype=torch.bfloat16, device="cuda")
    plan = P().VgemmPlan(dims, mm, nn, kk)
    P().vgemm(ta, tb, dims, out=c, plan=plan)  # warm-up (function attributes, tensor-map encoder)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        P().vgemm(ta, tb, dims, out=c, plan=plan)
    a2 = synth.round_bf16(synth.normal((4, mm, kk), 33))
    ta.copy_(bf16_cuda(a2))
    c.zero_()
    g.replay()
    torch.cuda.synchronize()
    ref = oracle.vgemm(a2, b, dims)
    got = to_np(c)
    for i, (m, n, k) in enumerate(dims):
        if m and n:
            assert rel_err(got[i, :m, :n], ref[i]) <= TOL_BF16


def test_vgemm_rejects_partial_k_block_inside_padding():
    a = bf16_cuda(np.zeros((2, 64, 128)))
    b = bf16_cuda(np.zeros((2, 128, 64)))
    with pytest.raises(Exception):
        P().vgemm(a, b, [(64, 64, 100), (64, 64, 128)])


@pytest.mark.parametrize("n,nc", [(128, 256), (384, 64), (1000, 264), (2048, 512)])
def test_trmm_parity_upper_triangle_ignored(n, nc):
    l = synth.round_bf16(synth.normal((n, n), 21) / np.sqrt(n))
    l_garbage = l.copy()
    l_garbage[np.triu_indices(n, 1)] = 1e4  # must never be read
    b = synth.round_bf16(synth.normal((n, nc), 22))
    c = to_np(P().trmm(bf16_cuda(l_garbage), bf16_cuda(b)))
    assert rel_err(c, oracle.trmm(l, b)) <= TOL_BF16


def test_trmm_identity_is_exact():
    n = 512
    b = synth.round_bf16(synth.normal((n, 256), 23))
    c = to_np(P().trmm(bf16_cuda(np.eye(n)), bf16_cuda(b)))
    np.testing.assert_array_equal(c, b)
