"""Pins P5-P9 of the SCW oracle and the test-error metric.  CPU only."""
import numpy as np
import pytest

import datagen
from oracle import scw, tucker1, validators


def _rand_rows(rng, k, m):
    q, _ = np.linalg.qr(rng.standard_normal((m, k)))
    return q.T


def test_p5_exactly_low_rank_gives_zero_error():
    """P5 (PAPER.md:149-153 with eps = 0): noise-free rank-p stream with a fixed
    column space, p <= r <= k: the trained S contains that space and SCW is exact."""
    c = datagen.lowrank("C1", rank=5)
    A_tr = datagen.generate(c, "train").numpy()
    A_te = datagen.generate(c, "test").numpy()
    S, lam, _ = tucker1.tucker1_sketch(A_tr, c.k)
    assert lam[5] <= 1e-10 * lam[0]          # exact rank 5
    for A in A_te:
        # the fp32 storage of a rank-5 matrix is rank 5 only up to fp32 rounding (~6e-8)
        e = scw.scw_error(A, S, c.r)
        eo = scw.best_rank_r_error(A, c.r)
        assert e <= 1e-6 * np.linalg.norm(A)
        assert eo <= 1e-6 * np.linalg.norm(A)


def test_p6_square_orthogonal_sketch_is_optimal():
    """P6: k = m (S orthogonal) gives SCW = [A]_r."""
    rng = np.random.default_rng(3)
    for (m, n, r) in [(12, 9, 3), (8, 20, 5), (30, 30, 1)]:
        A = rng.standard_normal((m, n))
        S = _rand_rows(rng, m, m)
        np.testing.assert_allclose(scw.scw(A, S, r), scw.best_rank_r(A, r), atol=1e-10)
        assert scw.scw_error(A, S, r) == pytest.approx(scw.best_rank_r_error(A, r), rel=1e-10)


def test_p6_topk_left_singular_sketch_is_optimal():
    """S = U_k(A)^T with k >= r gives [A]_r."""
    rng = np.random.default_rng(4)
    A = rng.standard_normal((20, 15))
    U = np.linalg.svd(A)[0]
    for k in (4, 6, 15):
        assert scw.scw_error(A, U[:, :k].T, 4) == pytest.approx(scw.best_rank_r_error(A, 4), rel=1e-10)


def test_p7_eckart_young_lower_bound_and_identity():
    """P7: e >= e_opt; and the proof identity
    ||A - [AV]_r V^T||^2 = ||A||^2 - ||[AV]_r||^2, i.e. e^2 = ||A||^2 - sum_{i<=r} sigma_i(AV)^2."""
    rng = np.random.default_rng(11)
    for _ in range(30):
        m, n = rng.integers(6, 25, size=2)
        k = int(rng.integers(2, m + 1))
        r = int(rng.integers(1, k + 1))
        A = rng.standard_normal((m, n))
        S = _rand_rows(rng, k, m)
        e = scw.scw_error(A, S, r)
        assert e >= scw.best_rank_r_error(A, r) - 1e-9 * np.linalg.norm(A)
        L, sig, R = scw.scw_factors(A, S, r)
        assert e ** 2 == pytest.approx(np.sum(A ** 2) - np.sum(sig ** 2), rel=1e-8, abs=1e-9 * np.sum(A ** 2))
        np.testing.assert_allclose(R.T @ R, np.eye(R.shape[1]), atol=1e-10)
        assert np.linalg.matrix_rank(L @ R.T) <= r


def test_scw_is_best_rank_r_in_rowspace():
    """Brute force: no random rank-r B with rowspace(B) in rowspace(SA) beats SCW."""
    rng = np.random.default_rng(12)
    A = rng.standard_normal((10, 8))
    S = _rand_rows(rng, 5, 10)
    r = 2
    e = scw.scw_error(A, S, r)
    V = np.linalg.svd(S @ A, full_matrices=False)[2].T
    for _ in range(300):
        X = rng.standard_normal((10, r)) @ rng.standard_normal((r, V.shape[1]))
        assert np.linalg.norm(A - X @ V.T) >= e - 1e-12
    # and local perturbations of the optimum in that class do not improve it
    L, _, R = scw.scw_factors(A, S, r)
    for _ in range(100):
        dL = 1e-3 * rng.standard_normal(L.shape)
        assert np.linalg.norm(A - (L + dL) @ R.T) >= e - 1e-12


def test_r_clamped_to_k():
    rng = np.random.default_rng(1)
    A = rng.standard_normal((9, 7))
    S = _rand_rows(rng, 3, 9)
    assert scw.scw_error(A, S, 5) == pytest.approx(scw.scw_error(A, S, 3), rel=1e-12)


def test_p8_theorem1_relaxation():
    """P8: sum_d ||A_d - SCW(A_d,S,r)||^2 <= ||A||^2 - ||[S A_(1)]_r||^2
    for any row-orthonormal S with k > r; with the Tucker1 S as well."""
    rng = np.random.default_rng(21)
    for _ in range(40):
        A = rng.standard_normal((5, 12, 9))
        S = _rand_rows(rng, 6, 12)
        lhs = float(np.sum(scw.scw_errors(A, S, 3) ** 2))
        assert lhs <= validators.theorem1_bound(A, S, 3) * (1 + 1e-12)
    A = datagen.generate("C1", "train").numpy()
    S, _, G = tucker1.tucker1_sketch(A, 10)
    lhs = float(np.sum(scw.scw_errors(A, S, 5) ** 2))
    rhs = validators.theorem1_bound(A, S, 5)
    assert lhs <= rhs * (1 + 1e-12)
    a = A.astype(np.float64)
    assert validators.theorem1_bound_from_gram(G, float(np.sum(a * a)), S, 5) == pytest.approx(rhs, rel=1e-9)


def test_p9_theorem2():
    """P9 (proof P:436-441): e^2 - e_opt^2 <= ||U_k U_k^T - S^T S||_F^2 ||A||_F^2."""
    rng = np.random.default_rng(31)
    for t in range(60):
        A = rng.standard_normal((14, 11))
        k, r = 6, 3
        U = np.linalg.svd(A)[0][:, :k]
        noise = rng.standard_normal((14, k)) * (10.0 ** -rng.integers(0, 4))
        S = np.linalg.qr(U + noise)[0].T
        e = scw.scw_error(A, S, r)
        eo = scw.best_rank_r_error(A, r)
        eps, a2 = validators.theorem2_gap(A, S, k, r)
        assert e ** 2 - eo ** 2 <= eps * a2 + 1e-10 * a2
    # eps = 0 case: S spans U_k exactly -> excess 0
    A = rng.standard_normal((14, 11))
    U = np.linalg.svd(A)[0][:, :6]
    eps, _ = validators.theorem2_gap(A, U.T, 6, 3)
    assert eps < 1e-20 * 100
    assert scw.scw_error(A, U.T, 3) == pytest.approx(scw.best_rank_r_error(A, 3), rel=1e-10)


def test_test_error_metric():
    """PAPER.md:248-252 and SPEC S:445-447 examples."""
    assert scw.test_error([0.0, 0.0], [1.0, 2.0])[0] == pytest.approx(-1.0)
    assert scw.test_error([1.02, 2.08], [1.0, 2.0])[0] == pytest.approx(0.03)
    assert scw.test_error([3.0, 4.0], [3.0, 4.0])[0] == 0.0
    mean, deg = scw.test_error([0.0, 5.0, 1.1], [0.0, 0.0, 1.0])
    assert deg == 1 and mean == pytest.approx(0.05)


def test_identical_slices_end_to_end():
    """SPEC S:454 / PAPER.md:147: train on copies of A, test on A, k >= r -> error = optimum."""
    rng = np.random.default_rng(8)
    A = rng.standard_normal((16, 12))
    S, _, _ = tucker1.tucker1_sketch(np.stack([A] * 5), 6)
    assert scw.scw_error(A, S, 4) == pytest.approx(scw.best_rank_r_error(A, 4), rel=1e-9)
