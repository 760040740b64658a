"""Pins of the Newton-Schulz / Muon oracle (R18)."""
import numpy as np
import pytest

from oracle import muon


@pytest.mark.parametrize("shape", [(37, 11), (11, 37), (64, 64), (200, 8)])
def test_ns_equals_svd_scalar_map(shape):
    """NS maps singular values through p^5 and keeps the singular vectors:
    NS(G) = U p^5(Sigma / ||G||_F) V^T (numpy SVD, an independent library route)."""
    G = np.random.default_rng(sum(shape)).standard_normal(shape)
    U, S, Vt = np.linalg.svd(G, full_matrices=False)
    ref = (U * muon.ns_scalar_map(S / (np.linalg.norm(G) + muon.NS_EPS))) @ Vt
    np.testing.assert_allclose(muon.newton_schulz(G), ref, atol=1e-10)


def test_ns_singular_values_band():
    """The Muon quintic does not converge to 1: five steps send every normalised
    singular value in [0.03, 1] into about [0.68, 1.14] (dense sampling of the scalar
    polynomial; SPEC's diag(3, 1) example lands in [0.7, 1.3]). The SPEC's
    "X^T X ~ I within 0.3" does not hold for this polynomial (R18)."""
    s = muon.ns_scalar_map(np.linspace(0.03, 1.0, 20001))
    assert s.min() > 0.67 and s.max() < 1.15
    assert muon.ns_scalar_map(np.logspace(-7, 0, 200001)).max() < 1.22   # overshoot for tiny inputs
    sv = np.linalg.svd(muon.newton_schulz(np.diag([3.0, 1.0])), compute_uv=False)
    assert np.all((sv > 0.7) & (sv < 1.3)), sv
    X = muon.newton_schulz(np.random.default_rng(3).standard_normal((8, 4)))
    sv = np.linalg.svd(X, compute_uv=False)
    assert np.all((sv > 0.67) & (sv < 1.15)), sv


def test_ns_scale_invariance_and_transpose():
    G = np.random.default_rng(5).standard_normal((30, 12))
    X = muon.newton_schulz(G)
    for c in (0.1, 10.0):
        np.testing.assert_allclose(muon.newton_schulz(c * G), X, atol=1e-6)
    np.testing.assert_allclose(muon.newton_schulz(G.T), X.T, atol=1e-12)


def test_ns_rejects_zero_and_bad_steps():
    with pytest.raises(ValueError):
        muon.newton_schulz(np.zeros((3, 3)))
    with pytest.raises(ValueError):
        muon.newton_schulz(np.ones((3, 3)), steps=0)


def test_muon_step_special_cases():
    """SPEC muon_step examples: lr = 0 leaves theta unchanged; zero gradient and zero
    momentum cannot be orthogonalised (rejected); weight decay alone scales theta."""
    rng = np.random.default_rng(7)
    th, g, m = rng.standard_normal((6, 4)), rng.standard_normal((6, 4)), np.zeros((6, 4))
    th2, m2 = muon.muon_step(th, g, m, lr=0.0)
    np.testing.assert_array_equal(th2, th)
    np.testing.assert_allclose(m2, g)
    th3, _ = muon.muon_step(th, g, m, lr=0.1, weight_decay=0.5, nesterov=False)
    np.testing.assert_allclose(th3, th * 0.95 - 0.1 * (6 / 4) ** 0.5 * muon.newton_schulz(g), atol=1e-12)


def test_muon_nesterov_branch_by_hand():
    """Nesterov look-ahead u = g + mu m' with m' = mu m + g (reading R18), pinned on a
    2 x 2 case worked by hand: mu = 0.5, g = diag(2/3, 0), m = diag(0, 4) give
    m' = diag(2/3, 2) and u = diag(2/3 + 1/3, 0 + 1) = I. The orthogonalisation of a
    multiple of the identity is a multiple of the identity (both singular values equal),
    so theta - theta' must be c*I with c in the quintic's band [0.67, 1.15] * lr.
    Every plausible slip breaks the proportionality: u = m' -> diag(2/3, 2); u = g + m'
    -> diag(4/3, 2); u = mu g + m' -> diag(1, 2); u = g + mu m -> diag(2/3, 2)."""
    g = np.diag([2.0 / 3.0, 0.0])
    m = np.diag([0.0, 4.0])
    th = np.array([[1.0, -2.0], [0.5, 3.0]])
    lr = 0.01
    th2, m2 = muon.muon_step(th, g, m, lr=lr, mu=0.5, nesterov=True)
    np.testing.assert_allclose(m2, np.diag([2.0 / 3.0, 2.0]), atol=1e-15)
    d = (th - th2) / lr
    assert abs(d[0, 1]) < 1e-12 and abs(d[1, 0]) < 1e-12
    assert d[0, 0] == pytest.approx(d[1, 1], rel=1e-12)
    assert 0.67 < d[0, 0] < 1.15
    # the plain-momentum branch on the same inputs orthogonalises diag(2/3, 2): unequal
    th3, m3 = muon.muon_step(th, g, m, lr=lr, mu=0.5, nesterov=False)
    np.testing.assert_allclose(m3, m2, atol=0)
    d3 = (th - th3) / lr
    assert abs(d3[0, 0] - d3[1, 1]) > 1e-3
