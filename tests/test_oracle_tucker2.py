"""Pins of the two-sided oracle (oracle/tucker2.py).  CPU only.

Each pin ties a function to something other than itself: the SVD of a single matrix
(Eckart-Young), exact multilinear-rank tensors, the Tucker1 closed form when l = n, the
one-sided SCW when W = I_n, and the stationarity conditions of Eq. (9) written through Grams
(a different computational route from the oracle's literal SVDs of unfoldings)."""
import numpy as np
import pytest

import datagen
from oracle import scw, tucker1, tucker2


def _orth_rows(rng, k, m):
    q, _ = np.linalg.qr(rng.standard_normal((m, k)))
    return q.T


def _multilinear(rng, D, m, n, k, l):
    U0 = np.linalg.qr(rng.standard_normal((m, k)))[0]
    V0 = np.linalg.qr(rng.standard_normal((n, l)))[0]
    return np.stack([U0 @ rng.standard_normal((k, l)) @ V0.T for _ in range(D)]), U0, V0


def test_unfoldings_and_mode2_gram():
    """A_(2) is n x mD and A_(2) A_(2)^T = sum_d A_d^T A_d; brute-force entry formula
    G2[j, j'] = sum_{d, i} A[d, i, j] A[d, i, j']."""
    rng = np.random.default_rng(0)
    A = rng.standard_normal((3, 4, 5))
    A2 = tucker2.mode2_unfold(A)
    assert A2.shape == (5, 12)
    G2 = tucker2.mode2_gram(A)
    brute = np.zeros((5, 5))
    for j in range(5):
        for jj in range(5):
            brute[j, jj] = sum(A[d, i, j] * A[d, i, jj] for d in range(3) for i in range(4))
    np.testing.assert_allclose(G2, brute, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(A2 @ A2.T, brute, rtol=1e-13, atol=1e-13)


def test_hooi_exact_multilinear_rank():
    """a tensor of exact multilinear rank (k, l, D) is reproduced (residual <=
    1e-8 ||t||) and span S = span U0, span W = span V0."""
    rng = np.random.default_rng(1)
    A, U0, V0 = _multilinear(rng, 6, 12, 9, 3, 2)
    S, W, hist, conv = tucker2.hooi_tucker2(A, 3, 2)
    assert hist[-1] <= 1e-8 * np.linalg.norm(A)
    assert tucker1.projector_distance(S, U0.T) <= 1e-8
    assert tucker1.projector_distance(W, V0.T) <= 1e-8


def test_hooi_single_slice_is_truncated_svd():
    """D' = 1, k = l = r: residual^2 = sum_{i>r} sigma_i(A)^2 (Eckart-Young)."""
    rng = np.random.default_rng(2)
    for (m, n, r) in [(10, 8, 3), (7, 12, 2), (15, 15, 5)]:
        A = rng.standard_normal((m, n))
        S, W, hist, _ = tucker2.hooi_tucker2(A[None], r, r)
        s = np.linalg.svd(A, compute_uv=False)
        assert hist[-1] ** 2 == pytest.approx(np.sum(s[r:] ** 2), rel=1e-8)


def test_hooi_residual_monotone():
    """SPEC S:255 / S:279: the residual history is non-increasing (slack 1e-9) on seeded
    random tensors, from the HOSVD init and from random initial factors."""
    rng = np.random.default_rng(3)
    for t in range(10):
        A = rng.standard_normal((4, 10, 8))
        S0 = _orth_rows(rng, 3, 10) if t % 2 else None
        W0 = _orth_rows(rng, 3, 8) if t % 2 else None
        _, _, hist, _ = tucker2.hooi_tucker2(A, 3, 3, max_iters=30, rel_tol=1e-14, S0=S0, W0=W0)
        assert all(b <= a + 1e-9 for a, b in zip(hist, hist[1:])), hist


def test_hooi_full_rank_one_sweep():
    """k = m, l = n reaches residual <= 1e-8 ||t|| in one sweep."""
    rng = np.random.default_rng(4)
    A = rng.standard_normal((5, 6, 4))
    _, _, hist, _ = tucker2.hooi_tucker2(A, 6, 4, max_iters=1)
    assert hist[1] <= 1e-8 * np.linalg.norm(A)


def test_hooi_with_l_equal_n_is_tucker1():
    """With l = n, W is orthogonal and the mode-1 step maximises ||S A_(1)||: S = Tucker1 S
    (the closed form of P:131 through G = sum A_d A_d^T)."""
    c = datagen.CONFIGS["C1"]
    A = datagen.generate(c, "train").numpy().astype(np.float64)
    S, W, _, _ = tucker2.hooi_tucker2(A, c.k, A.shape[2], max_iters=2)
    S1, lam, _ = tucker1.tucker1_sketch(A, c.k)
    assert tucker1.projector_distance(S, S1) <= 1e-8


def test_hooi_stationarity_through_grams():
    """At convergence S spans the top-k eigenvectors of sum_d A_d W^T W A_d^T and W the top-l
    eigenvectors of sum_d A_d^T S^T S A_d (eigh of explicit Grams, not SVDs of unfoldings),
    and the residual equals ||A||^2 - ||G||^2 (orthonormal factors, P:120-style identity)."""
    c = datagen.CONFIGS["C1"]
    A = datagen.generate(c, "train").numpy().astype(np.float64)
    k, l = c.k, 8
    S, W, hist, conv = tucker2.hooi_tucker2(A, k, l, max_iters=200, rel_tol=1e-13)
    G1 = sum(Ad @ W.T @ W @ Ad.T for Ad in A)
    G2 = sum(Ad.T @ S.T @ S @ Ad for Ad in A)
    S_g = np.linalg.eigh(G1)[1][:, ::-1][:, :k].T
    W_g = np.linalg.eigh(G2)[1][:, ::-1][:, :l].T
    assert tucker1.projector_distance(S, S_g) <= 1e-5
    assert tucker1.projector_distance(W, W_g) <= 1e-5
    core = tucker2.core(A, S, W)
    assert hist[-1] ** 2 == pytest.approx(np.sum(A * A) - np.sum(core * core), rel=1e-9)
    np.testing.assert_allclose(S @ S.T, np.eye(k), atol=1e-12)
    np.testing.assert_allclose(W @ W.T, np.eye(l), atol=1e-12)


def test_hooi_beats_hosvd_and_random_pairs():
    """Eq. (9): the HOOI objective ||G||^2 is >= the HOSVD init's and >= random orthonormal pairs'."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((6, 12, 10))
    S, W, hist, _ = tucker2.hooi_tucker2(A, 4, 3)
    e = tucker2.tucker2_residual(A, S, W)
    S0, W0 = tucker2.hosvd_init(A, 4, 3)
    assert e <= tucker2.tucker2_residual(A, S0, W0) + 1e-12
    for _ in range(20):
        assert e <= tucker2.tucker2_residual(A, _orth_rows(rng, 4, 12), _orth_rows(rng, 3, 10))


def test_two_sided_identity_sketches_give_best_rank_r():
    """SPEC S:349 / acceptance 1: S = I_m, W = I_n gives [A]_r; S = U_k^T, W = V_l^T also."""
    rng = np.random.default_rng(6)
    for (m, n, r) in [(12, 9, 3), (20, 30, 5), (8, 8, 1)]:
        A = rng.standard_normal((m, n))
        Ahat = tucker2.two_sided_scw(A, np.eye(m), np.eye(n), r)
        np.testing.assert_allclose(Ahat, scw.best_rank_r(A, r), atol=1e-10)
        U, s, Vt = np.linalg.svd(A)
        e = tucker2.two_sided_scw_error(A, U[:, :r + 2].T, Vt[:r + 1], r)
        assert e == pytest.approx(scw.best_rank_r_error(A, r), rel=1e-10)


def test_two_sided_bounds_and_identity():
    """For the same S, the two-sided approximation has its row space in span(Q) = rowspace(SA)
    and rank <= r, where SCW is the best such approximation, so e_opt <= e_one <= e_two; and
    e_two^2 = ||A||^2 - sum_{i<=r} sigma_i(P^T A Q)^2 (orthonormal P, Q)."""
    rng = np.random.default_rng(7)
    for _ in range(30):
        m, n = rng.integers(8, 25, size=2)
        k = int(rng.integers(2, m + 1))
        l = int(rng.integers(2, n + 1))
        r = int(rng.integers(1, min(k, l) + 1))
        A = rng.standard_normal((m, n))
        S, W = _orth_rows(rng, k, m), _orth_rows(rng, l, n)
        e2 = tucker2.two_sided_scw_error(A, S, W, r)
        e1 = scw.scw_error(A, S, r)
        eo = scw.best_rank_r_error(A, r)
        assert eo - 1e-9 <= e1 <= e2 + 1e-9
        _, sig, _ = tucker2.two_sided_scw_factors(A, S, W, r)
        assert e2 ** 2 == pytest.approx(np.sum(A * A) - np.sum(sig ** 2), rel=1e-9, abs=1e-9)


def test_two_sided_with_full_W_is_one_sided():
    """W = I_n (l = n): P spans col(A), so P [P^T A Q]_r Q^T = [AQ]_r Q^T = SCW(A, S, r)."""
    rng = np.random.default_rng(8)
    A = rng.standard_normal((14, 10))
    S = rng.standard_normal((5, 14))     # not orthonormal: Alg. 3 only uses its row space
    np.testing.assert_allclose(tucker2.two_sided_scw(A, S, np.eye(10), 3), scw.scw(A, S, 3), atol=1e-10)


def test_two_sided_exactly_low_rank():
    """Rank-p data (p <= r) with generic S, W (k, l >= p): rowspace(SA) = rowspace(A) and
    col(AW^T) = col(A), so the approximation is exact (e = 0)."""
    rng = np.random.default_rng(9)
    A = rng.standard_normal((20, 3)) @ rng.standard_normal((3, 16))
    S, W = rng.standard_normal((6, 20)), rng.standard_normal((5, 16))
    assert tucker2.two_sided_scw_error(A, S, W, 3) <= 1e-10 * np.linalg.norm(A)


def test_two_sided_trained_pair_identical_slices():
    """a pair trained on an identical-slice stream of A (k = l = r) captures A's
    top singular spaces exactly, so the two-sided error equals e_opt (P:147 analogue)."""
    rng = np.random.default_rng(10)
    A = rng.standard_normal((16, 12))
    S, W, _, _ = tucker2.hooi_tucker2(np.stack([A] * 4), 4, 4)
    assert tucker2.two_sided_scw_error(A, S, W, 4) == pytest.approx(scw.best_rank_r_error(A, 4), rel=1e-8)
