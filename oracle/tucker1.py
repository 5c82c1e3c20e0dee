"""Tucker1 sketch training, float64 (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

PAPER.md:116-131 (Section 3.1): the training loss (4)
    min_S sum_d ||A_d - S^T S A_d||_F^2  s.t.  S S^T = I_k
is equivalent (5)-(6) to max_S ||S A_(1)||_F^2, a Tucker1 decomposition along mode 1,
whose optimum is S* = (U^(1))_k^T, the first k left singular vectors of the mode-1
unfolding A_(1) = [A_1 | A_2 | ... | A_D'].  Since
A_(1) A_(1)^T = sum_d A_d A_d^T =: G, those are the top-k eigenvectors of G with
lambda_i(G) = sigma_i(A_(1))^2.  The oracle forms G (the plain sum) and calls eigh;
pin P1 (tests) checks it against the literal SVD of A_(1) on tiny inputs.

Readings:
* c3: the index formula of P:91 is garbled; only the block form of P:124 is used, and G
  does not depend on the column order of A_(1).
* c5: rows of S are ordered by decreasing eigenvalue; each row is sign-normalised so its
  entry of largest magnitude is positive (ties: lowest index).  S is compared across
  implementations through projectors / Ky Fan energy only.
"""
from __future__ import annotations

import numpy as np


def as_f64_stack(A) -> np.ndarray:
    """[D, m, n] float64 copy of the training stream (exact cast of the fp32 input)."""
    a = np.asarray(A)
    if a.ndim == 2:
        a = a[None]
    if a.ndim != 3:
        raise ValueError("expected a [D, m, n] stack of matrices")
    return a.astype(np.float64, copy=False)


def mode1_unfold(A) -> np.ndarray:
    """A_(1) = [A_1 | A_2 | ... | A_D]  (m x nD), the block form of PAPER.md:124."""
    a = as_f64_stack(A)
    return np.concatenate(list(a), axis=1)


def mode1_gram(A) -> np.ndarray:
    """G = sum_d A_d A_d^T  (m x m)  = A_(1) A_(1)^T."""
    a = as_f64_stack(A)
    G = np.zeros((a.shape[1], a.shape[1]), dtype=np.float64)
    for Ad in a:
        G += Ad @ Ad.T
    return G


def sign_normalise_rows(S: np.ndarray) -> np.ndarray:
    """Reading c5: the entry of largest |value| in each row is made positive
    (ties broken toward the lowest index, which np.argmax does)."""
    S = np.array(S, dtype=np.float64, copy=True)
    for i in range(S.shape[0]):
        j = int(np.argmax(np.abs(S[i])))
        if S[i, j] < 0:
            S[i] = -S[i]
    return S


def top_k_eigen(G: np.ndarray, k: int):
    """(S, lam): S = top-k eigenvectors of symmetric G as rows (k x m), lam = ALL
    eigenvalues of G in decreasing order."""
    G = np.asarray(G, dtype=np.float64)
    m = G.shape[0]
    if not (1 <= k <= m):
        raise ValueError(f"k={k} must satisfy 1 <= k <= m={m} (S is k x m, S S^T = I_k)")
    w, U = np.linalg.eigh(G)          # ascending
    order = np.argsort(w)[::-1]
    lam = w[order]
    S = U[:, order[:k]].T
    return sign_normalise_rows(S), lam


def tucker1_sketch(A, k: int):
    """Algorithm 2 lines 1-2: tensorise the training set, S <- Tucker1
    along mode 1.  Returns (S [k x m], lam [all eigenvalues of G, decreasing], G)."""
    G = mode1_gram(A)
    S, lam = top_k_eigen(G, k)
    return S, lam, G


def tucker1_sketch_svd(A, k: int):
    """The literal definition of: S* = first k columns of U^(1) (transposed)
    from the SVD A_(1) = U^(1) Sigma^(1) V^(1)T.  Brute force; tiny inputs only."""
    A1 = mode1_unfold(A)
    U, s, _ = np.linalg.svd(A1, full_matrices=False)
    return sign_normalise_rows(U[:, :k].T), s


def eigengap(lam: np.ndarray, k: int) -> float:
    """Reading c6: lambda_k / lambda_{k+1} (1-indexed, decreasing).  +inf when
    lambda_{k+1} == 0 < lambda_k; nan when lambda_k == 0 (undefined) or k == m."""
    lam = np.asarray(lam, dtype=np.float64)
    if k >= lam.size:
        return float("inf")
    lk, lk1 = lam[k - 1], lam[k]
    if lk <= 0:
        return float("nan")
    if lk1 <= 0:
        return float("inf")
    return float(lk / lk1)


def projector_distance(S1: np.ndarray, S2: np.ndarray) -> float:
    """||S1^T S1 - S2^T S2||_F  (projector form; reading c8)."""
    S1 = np.asarray(S1, dtype=np.float64)
    S2 = np.asarray(S2, dtype=np.float64)
    return float(np.linalg.norm(S1.T @ S1 - S2.T @ S2))


def kyfan_energy(G: np.ndarray, S: np.ndarray) -> float:
    """tr(S G S^T) = ||S A_(1)||_F^2, the objective of Eq. (5)."""
    S = np.asarray(S, dtype=np.float64)
    return float(np.trace(S @ np.asarray(G, dtype=np.float64) @ S.T))


def tucker1_loss(A, S) -> float:
    """Eq. (4): sum_d ||A_d - S^T S A_d||_F^2, evaluated directly."""
    a = as_f64_stack(A)
    S = np.asarray(S, dtype=np.float64)
    P = S.T @ S
    return float(sum(np.sum((Ad - P @ Ad) ** 2) for Ad in a))
