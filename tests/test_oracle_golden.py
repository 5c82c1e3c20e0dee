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
