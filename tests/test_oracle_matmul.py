"""Pins of the vgemm / trmm oracle against brute force and closed forms (CPU)."""
import numpy as np

import oracle
import synth


def _loop_matmul(a, b, m, n, k, lower_only=False):
    """Pure-Python MAC loops; lower_only: row i reduces over p <= i (the trmm vloop)."""
    c = [[0.0] * n for _ in range(m)]
    macs = 0
    for i in range(m):
        for j in range(n):
            acc = 0.0
            for p in range(k):
                if lower_only and p > i:
                    break
                acc += float(a[i][p]) * float(b[p][j])
                macs += 1
            c[i][j] = acc
    return np.array(c), macs


def test_vgemm_matches_loops_on_padded_buffers():
    dims = [(3, 5, 4), (1, 2, 7), (6, 1, 1), (0, 3, 2), (4, 4, 0)]
    mm, nn, kk = 6, 5, 7
    a = synth.normal((len(dims), mm, kk), 1)
    b = synth.normal((len(dims), kk, nn), 2)
    got = oracle.vgemm(a, b, dims)
    macs = 0
    for i, (m, n, k) in enumerate(dims):
        ref, mc = _loop_matmul(a[i], b[i], m, n, k)
        macs += mc
        assert got[i].shape == (m, n)
        np.testing.assert_allclose(got[i], ref.reshape(m, n), rtol=1e-12, atol=1e-12)
    assert 2 * macs == oracle.vgemm_flops(dims)


def test_vgemm_ignores_padding():
    dims = [(2, 3, 4)]
    a = synth.normal((1, 5, 6), 3)
    b = synth.normal((1, 6, 7), 4)
    a2, b2 = a.copy(), b.copy()
    a2[0, 2:, :] = np.nan   # padding rows of A
    a2[0, :, 4:] = np.nan   # padding columns of A
    b2[0, 4:, :] = np.nan
    b2[0, :, 3:] = np.nan
    np.testing.assert_array_equal(oracle.vgemm(a, b, dims)[0], oracle.vgemm(a2, b2, dims)[0])


def test_trmm_matches_vloop_and_ignores_upper_triangle():
    n, nc = 7, 3
    l = synth.normal((n, n), 5)
    b = synth.normal((n, nc), 6)
    ref, macs = _loop_matmul(l, b, n, nc, n, lower_only=True)
    np.testing.assert_allclose(oracle.trmm(l, b), ref, rtol=1e-12, atol=1e-12)
    assert 2 * macs == oracle.trmm_flops(n, nc)
    l2 = l.copy()
    l2[np.triu_indices(n, 1)] = 1e30  # never referenced
    np.testing.assert_array_equal(oracle.trmm(l, b), oracle.trmm(l2, b))


def test_trmm_special_cases():
    n = 9
    b = synth.normal((n, 4), 7)
    np.testing.assert_array_equal(oracle.trmm(np.eye(n), b), b)            # identity
    ones = np.ones((n, n))
    np.testing.assert_allclose(oracle.trmm(ones, b), np.cumsum(b, axis=0))  # tril(1) B = prefix sums


def test_padded_flop_ratio_and_workload_generator():
    d = synth.vgemm_dims(64, seed=1)
    assert d.shape == (64, 3) and d.min() >= 512 and d.max() <= 1408 and np.all(d % 128 == 0)
    dims = [tuple(map(int, r)) for r in d]
    assert oracle.vgemm_padded_flops(dims) >= oracle.vgemm_flops(dims)
    eq = [(512, 512, 512)] * 4
    assert oracle.vgemm_padded_flops(eq) == oracle.vgemm_flops(eq)
