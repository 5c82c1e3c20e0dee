"""Pins of the oracle against worked examples with hand-derived values (tests/golden/)."""
import numpy as np
import pytest

from oracle import scw, tucker1


def test_svd_2x2_rank1_error(golden):
    g = golden("svd_2x2.json")
    A = np.array(g["A"])
    assert scw.best_rank_r_error(A, 1) == pytest.approx(g["rank1_error"], rel=1e-13)
    assert abs(scw.best_rank_r_error(A, 1) - g["rank1_error_printed"]) < g["printed_tol"]
    # [A]_2 = A (full rank): zero error; [A]_1 has norm sigma_1
    assert scw.best_rank_r_error(A, 2) == pytest.approx(0.0, abs=1e-14)
    assert np.linalg.norm(scw.best_rank_r(A, 1)) == pytest.approx(g["sigma1"], rel=1e-13)


def test_mode1_unfold_and_gram(golden):
    g = golden("unfold_gram_2x2x2.json")
    slices = np.array(g["slices"])
    np.testing.assert_array_equal(tucker1.mode1_unfold(slices), np.array(g["mode1"]))
    np.testing.assert_array_equal(tucker1.mode1_gram(slices), np.array(g["gram"]))
    assert np.sum(slices ** 2) == g["fro_norm_sq"]


def test_tucker1_rank_one_slices(golden):
    g = golden("tucker1_e1.json")
    e1 = np.zeros((g["m"], g["n"]))
    e1[0, 0] = 1.0
    A = np.stack([e1] * g["D"])
    S, lam, G = tucker1.tucker1_sketch(A, g["k"])
    np.testing.assert_allclose(S[0], g["S_row0"], atol=1e-15)
    np.testing.assert_allclose(lam, g["eigenvalues"], atol=1e-14)
    np.testing.assert_allclose(S @ S.T, np.eye(g["k"]), atol=1e-14)


def test_scw_worked_example(golden):
    g = golden("scw_2x2.json")
    A = np.array(g["A"])
    S = np.array(g["S"])
    np.testing.assert_allclose(scw.scw(A, S, g["r"]), np.array(g["A_hat"]), rtol=1e-13)
    assert scw.scw_error(A, S, g["r"]) == pytest.approx(g["error"], rel=1e-13)
    # Eckart-Young: the sketched error cannot beat the optimum
    assert scw.scw_error(A, S, g["r"]) >= scw.best_rank_r_error(A, g["r"])


def test_projector_distance_spec_examples(golden):
    """SPEC S:106-109 worked examples of the projector distance (reading c8):
    U_k = e_1, S = e_2^T gives ||U_k U_k^T - S^T S||_F^2 = 2 (so the returned norm is sqrt 2);
    identical 2-dim subspaces of R^3 give 0.  The transposed form S S^T - U_k^T U_k of P:150 is
    1 x 1 (zero) on the first example and fails it."""
    g = golden("projector_e1_e2.json")
    Uk, S = np.array(g["U_k"]), np.array(g["S"])
    assert tucker1.projector_distance(Uk.T, S) ** 2 == pytest.approx(g["distance_sq"], rel=1e-15)
    assert tucker1.projector_distance(np.array(g["U_k_3"]).T, np.array(g["S_3"])) ** 2 == g["distance_sq_3"]
