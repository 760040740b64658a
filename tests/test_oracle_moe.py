"""Pins of the grouped-GEMM oracle: an independent one-hot
expert-assignment formulation, empty/ragged groups, argument checks."""
import numpy as np
import pytest

from oracle import moe


def test_grouped_mm_equals_onehot_einsum():
    rng = np.random.default_rng(0)
    G, N, K = 5, 7, 9
    sizes = np.array([3, 0, 6, 1, 4])
    off = np.concatenate([[0], np.cumsum(sizes)])
    a = rng.standard_normal((off[-1], K))
    b = rng.standard_normal((G, N, K))
    onehot = np.zeros((off[-1], G))
    onehot[np.arange(off[-1]), np.repeat(np.arange(G), sizes)] = 1.0
    ref = np.einsum("rg,gnk,rk->rn", onehot, b, a)      # select the expert by a one-hot, then contract
    np.testing.assert_allclose(moe.grouped_mm(a, b, off), ref, atol=1e-12)


def test_grouped_mm_single_group_is_a_matmul_and_checks_args():
    rng = np.random.default_rng(1)
    a, b = rng.standard_normal((6, 4)), rng.standard_normal((1, 3, 4))
    np.testing.assert_allclose(moe.grouped_mm(a, b, np.array([0, 6])), a @ b[0].T, atol=1e-12)
    with pytest.raises(ValueError):
        moe.grouped_mm(a, b, np.array([0, 5]))
    with pytest.raises(ValueError):
        moe.grouped_mm(a, np.concatenate([b, b]), np.array([0, 4, 3]))


def test_max_violation():
    """Balanced load -> 0; one expert with twice the mean... (PAPER.md L204 definition)."""
    assert moe.max_violation(np.full(8, 5.0)) == 0.0
    assert moe.max_violation(np.array([1.0, 1.0, 1.0, 5.0])) == pytest.approx(1.5)
    # every token on one of G experts: max = G * mean -> G - 1 (catches a max/mean swap or a
    # missing "- mean")
    assert moe.max_violation(np.array([0.0, 0.0, 12.0, 0.0, 0.0, 0.0])) == pytest.approx(5.0)


def test_rmsnorm_unit_mean_square_and_scale_invariance():
    x = np.random.default_rng(2).standard_normal((5, 64)) * 3.0
    y = moe.rmsnorm(x, np.ones(64), eps=0.0)
    np.testing.assert_allclose((y * y).mean(axis=1), 1.0, atol=1e-12)
    np.testing.assert_allclose(moe.rmsnorm(7.5 * x, np.ones(64), eps=0.0), y, atol=1e-12)
    g = np.linspace(0.5, 2.0, 64)
    np.testing.assert_allclose(moe.rmsnorm(x, g, eps=0.0), y * g, atol=1e-12)
