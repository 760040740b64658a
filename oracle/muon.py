"""fp64 oracle of Muon's Newton-Schulz orthogonalisation and update (TEST INFRASTRUCTURE).

PAPER.md §2.1.7 (L174-181): "Muon operates at the matrix level ... its Newton-Schulz
update requires access to the full gradient tensor"; the RL run uses Muon with lr
1e-6 (L440). The paper gives no iteration details; SPEC.md (S:L158-175,
newton_schulz_orthogonalize, muon_step) fixes the readings used here (R18):

  X_0     = G / ||G||_F                                      (Frobenius pre-normalisation)
  X_{j+1} = a X_j + b (X_j X_j^T) X_j + c (X_j X_j^T)^2 X_j   (quintic, (a, b, c) below)
  5 steps by default.

For a tall G (rows > cols) the same polynomial is applied through the Gram of the
columns, X_{j+1} = X_j (a I + b A + c A^2) with A = X_j^T X_j, which is the same
matrix (X X^T X = X (X^T X)). Either way every singular value sigma of X_0 is mapped
through p(s) = a s + b s^3 + c s^5, and the singular vectors are kept.

Muon step (reading R18): m <- mu m + g;  u = g + mu m (Nesterov) or m;
theta <- theta (1 - lr wd) - lr sqrt(max(1, rows/cols)) NS(u).
"""
from __future__ import annotations

import numpy as np

NS_COEFFS = (3.4445, -4.7750, 2.0315)   # the quintic of the Muon reference implementation
NS_EPS = 1e-7


def newton_schulz(G: np.ndarray, steps: int = 5, coeffs=NS_COEFFS) -> np.ndarray:
    """Newton-Schulz orthogonalisation in fp64, step by step (module docstring)."""
    G = np.asarray(G, dtype=np.float64)
    if steps < 1:
        raise ValueError("steps must be >= 1")
    nrm = np.linalg.norm(G)
    if nrm == 0.0:
        raise ValueError("zero matrix")
    a, b, c = coeffs
    X = G / (nrm + NS_EPS)
    tall = X.shape[0] > X.shape[1]
    for _ in range(steps):
        if tall:
            A = X.T @ X
            X = X @ (a * np.eye(A.shape[0]) + b * A + c * (A @ A))
        else:
            A = X @ X.T
            X = (a * np.eye(A.shape[0]) + b * A + c * (A @ A)) @ X
    return X


def ns_scalar_map(sigma: np.ndarray, steps: int = 5, coeffs=NS_COEFFS) -> np.ndarray:
    """p applied `steps` times to singular values (already normalised)."""
    a, b, c = coeffs
    s = np.asarray(sigma, dtype=np.float64)
    for _ in range(steps):
        s = a * s + b * s ** 3 + c * s ** 5
    return s


def muon_step(theta, grad, momentum, lr, mu=0.95, weight_decay=0.0, nesterov=True, steps=5):
    """One Muon update (reading R18); returns (theta', momentum')."""
    m = mu * np.asarray(momentum, np.float64) + np.asarray(grad, np.float64)
    u = np.asarray(grad, np.float64) + mu * m if nesterov else m
    rows, cols = u.shape
    scale = max(1.0, rows / cols) ** 0.5
    th = np.asarray(theta, np.float64) * (1.0 - lr * weight_decay) - lr * scale * newton_schulz(u, steps)
    return th, m
