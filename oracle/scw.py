"""SCW low-rank approximation and its errors, float64 (TEST INFRASTRUCTURE ONLY).

Algorithm 1, for A (m x n), sketch S (k x m), target rank r:
    1: (~, ~, V^T) <- SVD of SA
    2: [AV]_r      <- truncated rank-r SVD of AV
    3: A_hat       <- [AV]_r V^T

Readings:
* c1: V is the THIN n x k right factor (P:208 states AV in R^{m x k}; the proof of
  Theorem 1 uses Q in R^{n x k}).  When k > n the thin factor is n x n.
* c2: when rank(SA) < k numpy completes V with arbitrary orthonormal vectors; A_hat
  can then differ only by components of A along those completions, and the test
  data here always gives full-rank SA except in the exactly-low-rank pin, where
  A V_completion = 0 and A_hat is unchanged.
* c7: 1 <= r <= k <= m; r > k is clamped to k (SPEC S:381 behaviour).
* The error is the dense residual ||A - A_hat||_F (not ||A||^2 - sum sigma^2, which is
  equal in exact arithmetic, P:375 / P:422, and is used only as a pin).
"""
from __future__ import annotations

import numpy as np


def _f64(x) -> np.ndarray:
    return np.asarray(x, dtype=np.float64)


def scw_factors(A, S, r: int):
    """Algorithm 1 as factors: returns (L, sigma, R) with A_hat = L R^T, where
    L = U2_r diag(sigma_r) (m x r) and R = V W2_r (n x r) has orthonormal columns.
    (U2, sigma, W2^T) is the SVD of AV."""
    A = _f64(A)
    S = _f64(S)
    k, m = S.shape
    if A.shape[0] != m:
        raise ValueError("S is k x m and A must be m x n")
    r = min(int(r), k)
    if r < 1:
        raise ValueError("r must be >= 1")
    # line 1: V^T from the SVD of SA (thin; reading c1)
    _, _, Vt = np.linalg.svd(S @ A, full_matrices=False)
    V = Vt.T
    # line 2: truncated rank-r SVD of AV
    AV = A @ V
    U2, s2, W2t = np.linalg.svd(AV, full_matrices=False)
    r = min(r, s2.size)
    L = U2[:, :r] * s2[:r]
    R = V @ W2t[:r].T
    return L, s2[:r], R


def scw(A, S, r: int) -> np.ndarray:
    """A_hat = [AV]_r V^T (Algorithm 1, line 3)."""
    L, _, R = scw_factors(A, S, r)
    return L @ R.T


def scw_error(A, S, r: int) -> float:
    """||A - SCW(A, S, r)||_F, dense residual."""
    A = _f64(A)
    return float(np.linalg.norm(A - scw(A, S, r)))


def scw_errors(A_stack, S, r: int) -> np.ndarray:
    """Per-matrix SCW errors for a [B, m, n] stack."""
    return np.array([scw_error(A, S, r) for A in np.asarray(A_stack)], dtype=np.float64)


def best_rank_r_error(A, r: int) -> float:
    """||A - [A]_r||_F = sqrt(sum_{i>r} sigma_i(A)^2)  (Eckart-Young)."""
    s = np.linalg.svd(_f64(A), compute_uv=False)
    return float(np.sqrt(np.sum(s[r:] ** 2)))


def best_rank_r(A, r: int) -> np.ndarray:
    """[A]_r, the truncated rank-r SVD of A."""
    U, s, Vt = np.linalg.svd(_f64(A), full_matrices=False)
    return (U[:, :r] * s[:r]) @ Vt[:r]


def test_error(errors, errors_opt, degenerate_tol: float = 1e-12):
    """mean over the test set of (||A - A_hat|| - ||A - A_opt||) /
    ||A - A_opt||.  Reading c13: a matrix with ||A - A_opt|| = 0 contributes
    0 if its error is <= degenerate_tol, else it is excluded and counted as degenerate.
    Returns (mean, n_degenerate)."""
    e = _f64(errors)
    eo = _f64(errors_opt)
    terms = []
    n_deg = 0
    for a, b in zip(e, eo):
        if b == 0.0:
            if a <= degenerate_tol:
                terms.append(0.0)
            else:
                n_deg += 1
        else:
            terms.append((a - b) / b)
    mean = float(np.mean(terms)) if terms else float("nan")
    return mean, n_deg
