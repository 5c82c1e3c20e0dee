"""Pins of the matrix-free sketch oracle (oracle/matrix_free.py).  CPU only.

Each pin ties the randomized block Krylov oracle to something other than itself: the Gram formed
explicitly (a different route from the slice-wise products), the exact Tucker1 sketch when the
subspace is the whole space or contains range(A_(1)) (closed forms), Cauchy interlacing of Ritz
values (theta_i <= lambda_i), the nesting of Krylov spaces (more power steps never lower a Ritz
value, and block Krylov dominates subspace iteration from the same start), the Galerkin condition
of Rayleigh-Ritz, and scale invariance."""
import numpy as np
import pytest

import datagen
from oracle import matrix_free as mf
from oracle import tucker1


def _stack(seed, D, m, n):
    return np.random.default_rng(seed).standard_normal((D, m, n))


def _c1_planted(gap):
    c = datagen.planted("C1", gap=gap)
    return datagen.generate(c, "train").numpy().astype(np.float64), c


def test_g_times_equals_explicit_gram():
    """G Q from the slices equals (sum_d A_d A_d^T) Q with G formed explicitly."""
    A = _stack(1, 6, 9, 5)
    Q = np.random.default_rng(2).standard_normal((9, 4))
    G = np.zeros((9, 9))
    for d in range(6):
        for i in range(9):
            for j in range(9):
                G[i, j] += sum(A[d, i, t] * A[d, j, t] for t in range(5))
    np.testing.assert_allclose(mf.g_times(A, Q), G @ Q, rtol=1e-12, atol=1e-12)


def test_full_space_is_exact_tucker1():
    """p = m, q = 0: span(K) = R^m, so Rayleigh-Ritz IS the eigendecomposition of G: S equals the
    Tucker1 sketch and theta all eigenvalues."""
    A = _stack(3, 5, 12, 7)
    S0, lam, _ = tucker1.tucker1_sketch(A, 4)
    S, theta, K = mf.matrix_free_sketch(A, 4, datagen.start_block(12, 12, 0).numpy(), 0)
    assert K.shape == (12, 12)
    np.testing.assert_allclose(theta, lam, rtol=1e-10, atol=1e-10 * lam[0])
    assert tucker1.projector_distance(S, S0) < 1e-9


@pytest.mark.parametrize("krylov", [True, False])
def test_low_rank_stream_is_exact_after_one_step(krylov):
    """Exactly rank-rho stream (A_d = U0 C_d V_d^T, rho <= p): after one power step span(Q_1) =
    range(A_(1)) = range(U0), so the top-k Ritz pairs are the exact eigenpairs of G."""
    rng = np.random.default_rng(4)
    m, n, D, rho, k, p = 40, 30, 8, 6, 4, 8
    U0 = np.linalg.qr(rng.standard_normal((m, rho)))[0]
    A = np.stack([U0 @ rng.standard_normal((rho, n)) for _ in range(D)])
    S0, lam, _ = tucker1.tucker1_sketch(A, k)
    S, theta, _ = mf.matrix_free_sketch(A, k, datagen.start_block(m, p, 1).numpy(), 1, krylov)
    np.testing.assert_allclose(theta[:rho], lam[:rho], rtol=1e-10)
    assert tucker1.projector_distance(S, S0) < 1e-8


@pytest.mark.parametrize("q,krylov", [(0, True), (1, True), (3, True), (2, False)])
def test_cauchy_interlacing(q, krylov):
    """theta_i <= lambda_i(G) for every Ritz value (Cauchy interlacing for an orthonormal K), so the
    Ky Fan energy of S never exceeds the optimum sum_{i<=k} lambda_i."""
    A = _stack(5, 10, 30, 20)
    lam = tucker1.top_k_eigen(tucker1.mode1_gram(A), 1)[1]
    S, theta, K = mf.matrix_free_sketch(A, 5, datagen.start_block(30, 6, 2).numpy(), q, krylov)
    np.testing.assert_allclose(K.T @ K, np.eye(K.shape[1]), atol=1e-12)
    assert np.all(theta <= lam[: theta.size] * (1 + 1e-12) + 1e-12 * lam[0])
    assert tucker1.kyfan_energy(tucker1.mode1_gram(A), S) <= lam[:5].sum() * (1 + 1e-12)


def test_krylov_spaces_nest():
    """span K_q (block Krylov) contains span K_{q-1} and the subspace-iteration block Q_q from the
    same start, so every Ritz value is at least as large (interlacing on nested spaces)."""
    A = _stack(6, 10, 40, 25)
    om = datagen.start_block(40, 6, 3).numpy()
    prev = None
    for q in range(4):
        _, th, _ = mf.matrix_free_sketch(A, 5, om, q)
        _, th_sub, _ = mf.matrix_free_sketch(A, 5, om, q, krylov=False)
        assert np.all(th[:6] >= th_sub[:6] * (1 - 1e-12))
        if prev is not None:
            assert np.all(th[: prev.size] >= prev * (1 - 1e-12))
        prev = th


def test_ritz_values_and_galerkin_condition():
    """theta = eigvalsh(K^T G K) with G formed explicitly, and the residuals G x_i - theta_i x_i are
    orthogonal to span(K) (Rayleigh-Ritz / Galerkin condition)."""
    A = _stack(7, 6, 25, 15)
    G = tucker1.mode1_gram(A)
    S, theta, K = mf.matrix_free_sketch(A, 4, datagen.start_block(25, 5, 4).numpy(), 2)
    ref = np.sort(np.linalg.eigvalsh(K.T @ G @ K))[::-1]
    np.testing.assert_allclose(theta, ref, rtol=1e-10, atol=1e-12 * ref[0])
    for i in range(4):
        x = S[i]
        assert abs(np.linalg.norm(x) - 1) < 1e-12
        r = G @ x - (x @ G @ x) * x
        assert np.linalg.norm(K.T @ r) < 1e-9 * theta[0]
    np.testing.assert_allclose(np.sort(S @ G @ S.T, axis=None)[::-1][:1], theta[:1], rtol=1e-10)


def test_converges_to_tucker1_on_stream():
    """On the gap-planted C1 stream (lambda_k / lambda_{k+1} = 2.1), block Krylov with three steps
    reaches the exact Tucker1 subspace: projector distance and Ky Fan deficit at rounding level.
    (Krylov convergence goes with the gap: on the literal C1 stream, gap 1.16, the same run leaves a
    projector distance of ~1e-2 -- the method is an approximation, reading mf4.)"""
    A, c = _c1_planted(2.0)
    S0, lam, G = tucker1.tucker1_sketch(A, c.k)
    S, theta, _ = mf.matrix_free_sketch(A, c.k, datagen.start_block(c.m, c.k + 4, 5).numpy(), 3)
    assert tucker1.projector_distance(S, S0) < 1e-8
    np.testing.assert_allclose(theta[: c.k], lam[: c.k], rtol=1e-9)
    np.testing.assert_allclose(tucker1.kyfan_energy(G, S), lam[: c.k].sum(), rtol=1e-12)


def test_scale_invariance():
    """A -> 3A (no normalisation): same S, Ritz values scaled by 9."""
    A = _stack(8, 5, 20, 12)
    om = datagen.start_block(20, 6, 6).numpy()
    S1, t1, _ = mf.matrix_free_sketch(A, 4, om, 2)
    S2, t2, _ = mf.matrix_free_sketch(3.0 * A, 4, om, 2)
    np.testing.assert_allclose(t2, 9.0 * t1, rtol=1e-10)
    assert tucker1.projector_distance(S1, S2) < 1e-9


def test_rejects_bad_shapes():
    A = _stack(9, 2, 8, 4)
    with pytest.raises(ValueError):
        mf.matrix_free_sketch(A, 5, np.ones((8, 3)), 1)
    with pytest.raises(ValueError):
        mf.matrix_free_sketch(A, 2, np.ones((8, 3)), -1)
