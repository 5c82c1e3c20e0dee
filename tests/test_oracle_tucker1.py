"""Pins P1-P4, P10, P11 of the Tucker1 oracle.  CPU only."""
import numpy as np
import pytest

import datagen
from oracle import tucker1


def _rand_stack(seed, D, m, n):
    return np.random.default_rng(seed).standard_normal((D, m, n))


def _rand_rows(rng, k, m):
    q, _ = np.linalg.qr(rng.standard_normal((m, k)))
    return q.T


@pytest.mark.parametrize("D,m,n,k", [(5, 8, 6, 3), (20, 64, 48, 10), (3, 12, 20, 12), (7, 10, 3, 4)])
def test_p1_bruteforce_unfolding(D, m, n, k):
    """P1: eig(sum A_d A_d^T) has the same top-k subspace as the SVD
    of the explicit unfolding A_(1), and lambda_i = sigma_i(A_(1))^2."""
    A = _rand_stack(D * 1000 + m, D, m, n)
    S, lam, G = tucker1.tucker1_sketch(A, k)
    S_b, s = tucker1.tucker1_sketch_svd(A, k)
    r = min(m, n * D)
    np.testing.assert_allclose(lam[:r], s[:r] ** 2, rtol=1e-10, atol=1e-10 * lam[0])
    assert tucker1.projector_distance(S, S_b) < 1e-9
    # G equals A_(1) A_(1)^T computed from the unfolding
    A1 = tucker1.mode1_unfold(A)
    np.testing.assert_allclose(G, A1 @ A1.T, rtol=1e-12, atol=1e-12 * np.abs(G).max())


def test_p1_rowspace_single_slice_matches_svd():
    """D=1: S spans the top-k left singular vectors of the single matrix."""
    A = _rand_stack(3, 1, 9, 7)
    S, lam, _ = tucker1.tucker1_sketch(A, 4)
    U, s, _ = np.linalg.svd(A[0])
    assert tucker1.projector_distance(S, U[:, :4].T) < 1e-10
    np.testing.assert_allclose(lam[:7], s ** 2, rtol=1e-12)


def test_p2_kyfan_optimality():
    """P2 (Eq. (5)): tr(S G S^T) = sum_{i<=k} lambda_i >= tr(S' G S'^T)."""
    rng = np.random.default_rng(7)
    A = _rand_stack(11, 12, 16, 10)
    k = 5
    S, lam, G = tucker1.tucker1_sketch(A, k)
    best = tucker1.kyfan_energy(G, S)
    assert best == pytest.approx(lam[:k].sum(), rel=1e-12)
    for _ in range(50):
        Sp = _rand_rows(rng, k, 16)
        assert tucker1.kyfan_energy(G, Sp) <= best * (1 + 1e-12)
    # perturbing the optimum strictly decreases the energy (it is a maximiser)
    Sp = _rand_rows(np.random.default_rng(1), k, 16)
    mix = np.linalg.qr((S + 1e-2 * Sp).T)[0].T
    assert tucker1.kyfan_energy(G, mix) < best


def test_p3_loss_identity():
    """P3: sum_d ||A_d - S^T S A_d||^2 = ||A||^2 - ||S A_(1)||^2 for
    any row-orthonormal S, and the Tucker1 optimum minimises the loss (4)."""
    rng = np.random.default_rng(5)
    A = _rand_stack(5, 6, 14, 9)
    total = float(np.sum(A ** 2))
    for k in (1, 3, 7, 14):
        Sp = _rand_rows(rng, k, 14)
        G = tucker1.mode1_gram(A)
        assert tucker1.tucker1_loss(A, Sp) == pytest.approx(total - tucker1.kyfan_energy(G, Sp),
                                                            rel=1e-10, abs=1e-10 * total)
        S, lam, _ = tucker1.tucker1_sketch(A, k)
        assert tucker1.tucker1_loss(A, S) <= tucker1.tucker1_loss(A, Sp) + 1e-9 * total
        assert tucker1.tucker1_loss(A, S) == pytest.approx(total - lam[:k].sum(), rel=1e-9, abs=1e-9 * total)


def test_p4_identical_slices():
    """P4: if all A_d = A then span S = span U_k(A)."""
    A0 = _rand_stack(9, 1, 20, 15)[0]
    A = np.stack([A0] * 6)
    for k in (3, 8):
        S, _, _ = tucker1.tucker1_sketch(A, k)
        U = np.linalg.svd(A0)[0][:, :k]
        assert tucker1.projector_distance(S, U.T) < 1e-9


def test_p10_invariants_c1():
    """P10: G symmetric PSD, S S^T = I_k, rows sorted by eigenvalue, sign convention c5."""
    A = datagen.generate("C1", "train").numpy()
    S, lam, G = tucker1.tucker1_sketch(A, 10)
    np.testing.assert_array_equal(G, G.T)
    assert lam[-1] >= -1e-12 * lam[0]
    assert np.all(np.diff(lam) <= 0)
    np.testing.assert_allclose(S @ S.T, np.eye(10), atol=1e-13)
    for row in S:
        j = int(np.argmax(np.abs(row)))
        assert row[j] > 0
    # Rayleigh quotients of the rows are the top eigenvalues, in order
    np.testing.assert_allclose(np.diag(S @ G @ S.T), lam[:10], rtol=1e-10)


def test_p11_invariances():
    """P11: permuting the training order, splitting it into shards whose
    partial Grams are summed, or scaling the data by c > 0 leave span S unchanged."""
    A = datagen.generate("C1", "train").numpy().astype(np.float64)
    S, lam, G = tucker1.tucker1_sketch(A, 10)
    perm = np.random.default_rng(0).permutation(A.shape[0])
    S_p, _, G_p = tucker1.tucker1_sketch(A[perm], 10)
    assert tucker1.projector_distance(S, S_p) < 1e-9
    np.testing.assert_allclose(G_p, G, rtol=1e-12, atol=1e-12 * np.abs(G).max())
    for P in (2, 4, 8):
        Gs = sum(tucker1.mode1_gram(A[(p * 20) // P:((p + 1) * 20) // P]) for p in range(P))
        np.testing.assert_allclose(Gs, G, rtol=1e-12, atol=1e-12 * np.abs(G).max())
    for c in (1e-3, 7.0, 2.0 ** 20):
        S_c, lam_c, _ = tucker1.tucker1_sketch(c * A, 10)
        assert tucker1.projector_distance(S, S_c) < 1e-8
        np.testing.assert_allclose(lam_c[:10], c * c * lam[:10], rtol=1e-10)


def test_eigengap_reading_c6():
    assert tucker1.eigengap(np.array([4.0, 2.0, 1.0]), 1) == 2.0
    assert tucker1.eigengap(np.array([4.0, 0.0, 0.0]), 1) == float("inf")
    assert np.isnan(tucker1.eigengap(np.array([4.0, 0.0, 0.0]), 2))
    assert tucker1.eigengap(np.array([4.0, 2.0]), 2) == float("inf")


def test_k_out_of_range():
    with pytest.raises(ValueError):
        tucker1.top_k_eigen(np.eye(3), 4)
    with pytest.raises(ValueError):
        tucker1.top_k_eigen(np.eye(3), 0)


def test_projector_distance_principal_angles():
    """Projector distance (reading c8) against closed forms that do not use the
    projectors: for row-orthonormal k x m S1, S2, ||S1^T S1 - S2^T S2||_F^2 = 2k - 2||S1 S2^T||_F^2
    = 2 sum_i sin^2(angle_i); in the plane, lines at angle t are sqrt(2)|sin t| apart.  A transposed
    (k x k) or unsquared mutation fails every case."""
    for t in (0.0, 0.3, np.pi / 4, 1.2, np.pi / 2):
        S1 = np.array([[1.0, 0.0, 0.0]])
        S2 = np.array([[np.cos(t), np.sin(t), 0.0]])
        assert tucker1.projector_distance(S1, S2) == pytest.approx(np.sqrt(2) * abs(np.sin(t)), abs=1e-15)
    rng = np.random.default_rng(11)
    for k, m in ((1, 5), (3, 7), (4, 4), (6, 20)):
        S1, S2 = _rand_rows(rng, k, m), _rand_rows(rng, k, m)
        cos = np.linalg.svd(S1 @ S2.T, compute_uv=False)
        want = 2.0 * np.sum(1.0 - np.clip(cos, 0, 1) ** 2)
        assert tucker1.projector_distance(S1, S2) ** 2 == pytest.approx(want, rel=1e-10, abs=1e-12)
        # the same subspace in another basis: 0
        Q = np.linalg.qr(rng.standard_normal((k, k)))[0]
        assert tucker1.projector_distance(S1, Q @ S1) < 1e-13
    # nonzero value on a case the k x k form makes vanish
    assert tucker1.projector_distance(_rand_rows(rng, 2, 6), _rand_rows(rng, 2, 6)) > 0.1
