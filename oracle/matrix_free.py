"""Matrix-free Tucker1 sketch by randomized block Krylov, float64 (TEST INFRASTRUCTURE ONLY; see
oracle/__init__.py).

SURVEY.md §8(f) row f4 (second half): the sketch of Algorithm 2 line 2 (S <- Tucker1, PAPER.md:165,
i.e. the top-k left singular vectors of A_(1)) approximated WITHOUT forming the mode-1 Gram
G = A_(1) A_(1)^T = sum_d A_d A_d^T.  The paper names pass-efficiency as future work
 and the memory cost of the whole training tensor as a limitation; it gives no such
algorithm, so this follows the standard randomized block Krylov method (readings mf1-mf4 in
DESIGN.md), step by step:

  input  A_1..A_D (m x n), k, a start block Omega (m x p, p >= k), q >= 0 power steps
  1. Q_0 = orth(Omega)
  2. for j = 1..q:  Y_j = G Q_{j-1} = sum_d A_d (A_d^T Q_{j-1})           (two passes over A)
                    Krylov:   Y_j <- Y_j - sum_{i<j} Q_i Q_i^T Y_j, twice   (block Gram-Schmidt)
                              Q_j = orth(Y_j) minus the directions with singular value
                                    <= 1e-10 ||G Q_{j-1}||_2 (breakdown, reading mf3)
                              K = [Q_0 | ... | Q_q]     (m x (q+1)p at most)
                    subspace: Q_j = orth(Y_j);   K = Q_q                   (m x p)
  3. Rayleigh-Ritz on span(K) through one more pass:
        Z_d = A_d^T K,  H = sum_d Z_d^T Z_d  (= K^T G K)
        (theta, W) = eigh(H), decreasing;  X = K W[:, :k]
  4. S = X^T with the sign rule of reading c5; the Ritz values theta_1..theta_k stand in for the
     top-k eigenvalues of G.

orth(.) is numpy's reduced QR (any orthonormal basis of the same span gives the same Ritz pairs).
Only the A_d are touched, never G: the products use the slices as stored (P:124's block form).
"""
from __future__ import annotations

import numpy as np

from .tucker1 import as_f64_stack, sign_normalise_rows


def g_times(A, Q) -> np.ndarray:
    """G Q = sum_d A_d (A_d^T Q) without forming G (G = A_(1) A_(1)^T)."""
    a = as_f64_stack(A)
    Q = np.asarray(Q, dtype=np.float64)
    Y = np.zeros((a.shape[1], Q.shape[1]))
    for Ad in a:
        Y += Ad @ (Ad.T @ Q)
    return Y


def orth(Y) -> np.ndarray:
    """Orthonormal basis of range(Y) (reduced QR), m x p."""
    Q, _ = np.linalg.qr(np.asarray(Y, dtype=np.float64))
    return Q


def orth_deflated(Y, scale: float, rtol: float = 1e-10) -> np.ndarray:
    """Orthonormal basis of the numerically nonzero part of range(Y): left singular vectors with
    sigma > rtol * scale (reading mf3: block Krylov breakdown -- directions of the new block that
    the previous blocks already span are dropped, not kept as rounding noise)."""
    U, s, _ = np.linalg.svd(np.asarray(Y, dtype=np.float64), full_matrices=False)
    return U[:, s > rtol * scale]


def krylov_basis(A, Omega, q: int, krylov: bool = True) -> np.ndarray:
    """Steps 1-2: K = [Q_0 | ... | Q_q] (block Krylov) or Q_q (subspace iteration)."""
    if q < 0:
        raise ValueError("q >= 0")
    blocks = [orth(Omega)]
    for _ in range(q):
        Y = g_times(A, blocks[-1])
        if krylov:
            scale = np.linalg.norm(Y, 2)
            for _ in range(2):
                for B in blocks:
                    Y = Y - B @ (B.T @ Y)
            Qj = orth_deflated(Y, scale)
            if Qj.shape[1] == 0:  # span(K) is invariant under G: the Krylov space is exhausted
                break
            blocks.append(Qj)
        else:
            blocks = [orth(Y)]
    return np.hstack(blocks)


def rayleigh_ritz(A, K, k: int):
    """Step 3-4: (S [k x m], theta [all w Ritz values, decreasing]) from span(K) via
    H = sum_d (A_d^T K)^T (A_d^T K)."""
    a = as_f64_stack(A)
    K = np.asarray(K, dtype=np.float64)
    w = K.shape[1]
    if not (1 <= k <= w):
        raise ValueError(f"k={k} must satisfy 1 <= k <= width={w}")
    H = np.zeros((w, w))
    for Ad in a:
        Z = Ad.T @ K
        H += Z.T @ Z
    t, W = np.linalg.eigh(H)
    order = np.argsort(t)[::-1]
    theta = t[order]
    X = K @ W[:, order[:k]]
    return sign_normalise_rows(X.T), theta


def matrix_free_sketch(A, k: int, Omega, q: int, krylov: bool = True):
    """Steps 1-4.  Returns (S [k x m], theta [w], K [m x w])."""
    Omega = np.asarray(Omega, dtype=np.float64)
    if Omega.ndim != 2 or Omega.shape[1] < k:
        raise ValueError("Omega must be m x p with p >= k")
    K = krylov_basis(A, Omega, q, krylov)
    S, theta = rayleigh_ritz(A, K, k)
    return S, theta, K
