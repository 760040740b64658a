"""fp64 oracle of the MoE grouped GEMM (TEST INFRASTRUCTURE).

PAPER.md §2.1.8 (L183-200, Fig. 5): expert projections run as torch._grouped_mm
with hidden dim 4096 and MoE dim 1408; tokens routed to expert g occupy the rows
[offsets[g], offsets[g+1]) of the (permuted) activation matrix. Definition:

  out[r, :] = sum_k a[r, k] * b[g(r), n, k]      for r in [offsets[g], offsets[g+1])
"""
from __future__ import annotations

import numpy as np


def grouped_mm(a: np.ndarray, b: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    G, N, K = b.shape
    offsets = np.asarray(offsets, np.int64)
    if a.shape[1] != K or len(offsets) != G + 1 or offsets[0] != 0 or offsets[-1] != a.shape[0] \
            or np.any(np.diff(offsets) < 0):
        raise ValueError("bad grouped_mm arguments")
    out = np.empty((a.shape[0], N))
    for g in range(G):
        r0, r1 = offsets[g], offsets[g + 1]
        out[r0:r1] = a[r0:r1] @ b[g].T
    return out


def max_violation(expert_load: np.ndarray) -> float:
    """MaxViolation = (max_i Load_i - mean Load) / mean Load."""
    load = np.asarray(expert_load, np.float64)
    return float((load.max() - load.mean()) / load.mean())


def rmsnorm(x: np.ndarray, gamma: np.ndarray, eps: float = 1e-6) -> np.ndarray:
    """RMSNorm(x) = x / sqrt(mean(x^2) + eps) * gamma, per row (the pre-MoE norm)."""
    x = np.asarray(x, np.float64)
    return x / np.sqrt((x * x).mean(axis=1, keepdims=True) + eps) * np.asarray(gamma, np.float64)


def grouped_mm_rmsnorm(x, gamma, b, offsets, eps=1e-6) -> np.ndarray:
    """The expert projection of normalised tokens: grouped_mm(RMSNorm(x), b, offsets)."""
    return grouped_mm(rmsnorm(x, gamma, eps), b, offsets)
