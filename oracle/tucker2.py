"""Two-sided variant: Tucker2 by HOOI and two-sided SCW, float64 (TEST INFRASTRUCTURE ONLY;
see oracle/__init__.py).  SURVEY.md §8(f) row f1.

PAPER.md:178-187 (Section 3.2, Eq. (9)):
    min_{S, W, G} ||A - G x_1 S^T x_2 W^T||_F^2   s.t.  S S^T = I_k,  W W^T = I_l,
with no closed form; it is approximated by HOOI (Appendix Algorithm 5).
Algorithm 3, two-sided SCW, for a test matrix A (m x n):
    1: Q <- QR of A^T S^T          (n x k)
    2: P <- QR of A W^T            (m x l)
    3: [P^T A Q]_r <- truncated rank-r SVD of P^T A Q   (l x k)
    4: A_hat = P [P^T A Q]_r Q^T

Readings (f1 readings):
* t1: Tucker2 = Algorithm 5 over modes 1 and 2 only (the mode-3 factor is the identity,
  P:181 "Tucker2 ... along the mode-1 and 2"); the paper's unspecified "initial guess" is the
  HOSVD one: S0 = top-k left singular vectors of A_(1), W0 = top-l of A_(2).
* t2: Algorithm 5 updates the modes in order 1, 2 inside each sweep; the unfolding
  B_(n) of the projected tensor is formed in block form (P:124 style):
      mode 1: B_d = A_d W^T (m x l),  B_(1) = [B_1 | ... | B_D]          (m x lD)
      mode 2: C_d = S A_d   (k x n),  B_(2) = [C_1^T | ... | C_D^T]      (n x kD)
  (column order of an unfolding does not change its left singular vectors).
* t3: "while not convergent": stop when the relative change of the residual
  ||A - G x_1 S^T x_2 W^T||_F between sweeps is <= rel_tol, or after max_iters sweeps.
* t4: the core is G_d = S A_d W^T (Alg. 5 line 8 in tensor format); with orthonormal S, W the
  residual is computed directly as sum_d ||A_d - S^T G_d W||_F^2 (no identity shortcut).
* c5 applies to S and W: rows ordered by decreasing singular value, largest-|entry| positive.
* Algorithm 3's QR may be any orthonormal basis of the same column space (the factor
  is only used for orthogonalisation); the oracle uses numpy's Householder QR.
"""
from __future__ import annotations

import numpy as np

from .tucker1 import as_f64_stack, sign_normalise_rows


def mode2_unfold(A) -> np.ndarray:
    """A_(2) = [A_1^T | A_2^T | ... | A_D^T]  (n x mD): the mode-2 fibres (block form)."""
    a = as_f64_stack(A)
    return np.concatenate([Ad.T for Ad in a], axis=1)


def mode2_gram(A) -> np.ndarray:
    """sum_d A_d^T A_d  (n x n) = A_(2) A_(2)^T (BASELINE north_star's mode-2 Gram)."""
    a = as_f64_stack(A)
    G = np.zeros((a.shape[2], a.shape[2]), dtype=np.float64)
    for Ad in a:
        G += Ad.T @ Ad
    return G


def _top_left_singular(B: np.ndarray, k: int) -> np.ndarray:
    """Rows = first k left singular vectors of B (truncated rank-k SVD, Alg. 5 line 6)."""
    U, _, _ = np.linalg.svd(B, full_matrices=False)
    if U.shape[1] < k:  # rank-deficient / short unfolding: deterministic completion
        Q, _ = np.linalg.qr(np.concatenate([U, np.eye(B.shape[0])], axis=1))
        U = np.concatenate([U, Q[:, U.shape[1]:k]], axis=1)
    return sign_normalise_rows(U[:, :k].T)


def hosvd_init(A, k: int, l: int):
    """Reading t1: S0 = top-k left singular vectors of A_(1), W0 = top-l of A_(2)."""
    a = as_f64_stack(A)
    S0 = _top_left_singular(np.concatenate(list(a), axis=1), k)
    W0 = _top_left_singular(mode2_unfold(a), l)
    return S0, W0


def core(A, S, W) -> np.ndarray:
    """G_d = S A_d W^T  ([D, k, l]; Alg. 5 line 8 / Eq. (9))."""
    a = as_f64_stack(A)
    S = np.asarray(S, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    return np.stack([S @ Ad @ W.T for Ad in a])


def tucker2_residual(A, S, W) -> float:
    """||A - G x_1 S^T x_2 W^T||_F with G the projected core (reading t4), evaluated directly."""
    a = as_f64_stack(A)
    S = np.asarray(S, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    tot = 0.0
    for Ad in a:
        R = Ad - S.T @ (S @ Ad @ W.T) @ W
        tot += float(np.sum(R * R))
    return float(np.sqrt(tot))


def hooi_tucker2(A, k: int, l: int, max_iters: int = 100, rel_tol: float = 1e-8, S0=None, W0=None):
    """Algorithm 5 restricted to modes 1-2 (readings t1-t3).
    Returns (S [k x m], W [l x n], history [residual after the init and after each sweep], converged)."""
    a = as_f64_stack(A)
    D, m, n = a.shape
    if not (1 <= k <= m and 1 <= l <= n):
        raise ValueError(f"need 1 <= k <= m ({k}, {m}) and 1 <= l <= n ({l}, {n})")
    if S0 is None or W0 is None:
        Si, Wi = hosvd_init(a, k, l)
        S = Si if S0 is None else np.asarray(S0, dtype=np.float64)
        W = Wi if W0 is None else np.asarray(W0, dtype=np.float64)
    else:
        S, W = np.asarray(S0, dtype=np.float64), np.asarray(W0, dtype=np.float64)
    hist = [tucker2_residual(a, S, W)]
    converged = False
    for _ in range(max_iters):
        # mode 1: B = A x_2 W^T (W fixed at its current iterate), truncated SVD of B_(1)
        B1 = np.concatenate([Ad @ W.T for Ad in a], axis=1)
        S = _top_left_singular(B1, k)
        # mode 2: B = A x_1 S^T with the NEW S (Alg. 5 line 4: modes < n use U_{k+1})
        B2 = np.concatenate([(S @ Ad).T for Ad in a], axis=1)
        W = _top_left_singular(B2, l)
        hist.append(tucker2_residual(a, S, W))
        prev, cur = hist[-2], hist[-1]
        if abs(prev - cur) <= rel_tol * max(prev, np.finfo(float).tiny):
            converged = True
            break
    return S, W, hist, converged


def two_sided_scw_factors(A, S, W, r: int):
    """Algorithm 3 as factors: (L [m x r], sigma [r], R [n x r]) with A_hat = L R^T,
    L = P U_r diag(sigma_r), R = Q V_r, where U diag(sigma) V^T is the SVD of P^T A Q."""
    A = np.asarray(A, dtype=np.float64)
    S = np.asarray(S, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    if S.shape[1] != A.shape[0] or W.shape[1] != A.shape[1]:
        raise ValueError("S must be k x m and W l x n for an m x n A")
    Q, _ = np.linalg.qr(A.T @ S.T)     # line 1
    P, _ = np.linalg.qr(A @ W.T)       # line 2
    M = P.T @ A @ Q                    # line 3
    U, s, Vt = np.linalg.svd(M, full_matrices=False)
    r = min(int(r), s.size)
    L = (P @ U[:, :r]) * s[:r]
    R = Q @ Vt[:r].T
    return L, s[:r], R


def two_sided_scw(A, S, W, r: int) -> np.ndarray:
    """A_hat = P [P^T A Q]_r Q^T (Algorithm 3, line 4)."""
    L, _, R = two_sided_scw_factors(A, S, W, r)
    return L @ R.T


def two_sided_scw_error(A, S, W, r: int) -> float:
    """||A - two_sided_SCW(A, S, W, r)||_F, dense residual."""
    A = np.asarray(A, dtype=np.float64)
    return float(np.linalg.norm(A - two_sided_scw(A, S, W, r)))


def two_sided_scw_errors(A_stack, S, W, r: int) -> np.ndarray:
    return np.array([two_sided_scw_error(A, S, W, r) for A in np.asarray(A_stack)], dtype=np.float64)
