"""Executable forms of the paper's theorems (TEST INFRASTRUCTURE ONLY).

These need no oracle output: they hold for ANY row-orthonormal S, so they check
the GPU path (its S and its SCW errors) and the oracle alike.
"""
from __future__ import annotations

import numpy as np

from .tucker1 import as_f64_stack, mode1_unfold


def theorem1_bound(A_train, S, r: int) -> float:
    """Right-hand side of Eq. (7), PAPER.md:137-141:
        ||A||_F^2 - ||[S A_(1)]_r||_F^2,
    where ||[S A_(1)]_r||_F^2 = sum of the r largest squared singular values of S A_(1)
    = sum of the r largest eigenvalues of S G S^T (G = A_(1) A_(1)^T)."""
    a = as_f64_stack(A_train)
    S = np.asarray(S, dtype=np.float64)
    total = float(np.sum(a * a))
    SA1 = S @ mode1_unfold(a)
    s = np.linalg.svd(SA1, compute_uv=False)
    return total - float(np.sum(s[:r] ** 2))


def theorem1_bound_from_gram(G, A_fro2: float, S, r: int) -> float:
    """Same quantity from G (no unfolding): eig(S G S^T) are sigma_i(S A_(1))^2."""
    S = np.asarray(S, dtype=np.float64)
    mu = np.linalg.eigvalsh(S @ np.asarray(G, dtype=np.float64) @ S.T)[::-1]
    return float(A_fro2) - float(np.sum(mu[:r]))


def theorem2_gap(A, S, k: int, r: int):
    """Theorem 2 with the proof's constant (reading c8):
        ||A - SCW(A,S,r)||^2 - ||A - [A]_r||^2  <=  ||U_k U_k^T - S^T S||_F^2 ||A||_F^2.
    Returns (lhs_without_scw_error, rhs_factor) pieces: (eps, ||A||_F^2), where
    eps = ||U_k U_k^T - S^T S||_F^2 and U_k are the first k left singular vectors of A."""
    A = np.asarray(A, dtype=np.float64)
    S = np.asarray(S, dtype=np.float64)
    U, _, _ = np.linalg.svd(A, full_matrices=False)
    Uk = U[:, :k]
    eps = float(np.linalg.norm(Uk @ Uk.T - S.T @ S) ** 2)
    return eps, float(np.sum(A * A))
