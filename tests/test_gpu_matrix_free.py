"""Parity of the matrix-free Tucker1 sketch (randomized block Krylov) on the
GPU with the float64 oracle (oracle/matrix_free.py), through the C ABI.

Both sides start from the same seeded block Omega (datagen.start_block).  Tolerances, from the
arithmetic: every product with the slices is 3xTF32, whose dropped L*L term and truncating operand
read leave an error of ~2^-21 sum_i |a_i k_i| per entry of Z_d = A_d^T K (E2) -- relative to the
entry itself that is ~1e-6 once K holds directions of small energy -- and H = sum_d Z_d^T Z_d and a
Ritz value depend on those entries to first order -> |theta - theta_o| <= 1e-5 theta_1 and Ky Fan
within 1e-5 relative (measured 2.9e-6 at C1, a bias toward smaller |Z|); the subspace itself (projector of S) is compared only
where the Ritz gap at k is planted (>= 2), at 1e-4 (reading c16).  Interlacing theta_i <= lambda_i
(the exact eigenvalues of G) holds for any orthonormal K and is checked at every size.
"""
import numpy as np
import pytest
import torch

import datagen
import paper_2209_14637_b200 as tsk
from oracle import matrix_free as omf
from oracle import scw as oscw
from oracle import tucker1

pytestmark = pytest.mark.gpu


def _block(k, oversample, m):
    p = (k + oversample + 3) // 4 * 4
    return min(p, m)


def _run(A, k, oversample, q, subspace=False, seed=7):
    D, m, n = A.shape
    p = _block(k, oversample, m)
    om = datagen.start_block(m, p, seed)
    S, lam, info, st = tsk.sketch_train_matrix_free(A.cuda(), k, oversample=oversample, power_iters=q,
                                                    subspace=subspace, omega=om.cuda())
    So, th, K = omf.matrix_free_sketch(A.numpy(), k, om.numpy(), q, krylov=not subspace)
    return S.cpu().double().numpy(), lam.cpu().numpy(), info, st, So, th, K


@pytest.mark.parametrize("cfg,D,k,ov,q,subspace", [
    ("C1", None, 10, 4, 2, False),
    ("C1", None, 10, 10, 1, True),
    ("C2", 100, 20, 16, 2, False),
    ("C2", 60, 20, 8, 3, True),
    ("C3", 30, 40, 16, 2, False),
])
def test_matrix_free_matches_oracle(cfg, D, k, ov, q, subspace):
    c = datagen.CONFIGS[cfg]
    A = datagen.generate(c, "train", 0, D or c.D_train)
    S, lam, info, st, So, th, K = _run(A, k, ov, q, subspace)
    assert st == 0
    assert info["power_iters"] == q and info["width"] == K.shape[1] and info["passes"] == 2 * q + 1
    assert np.all(np.abs(lam - th[:k]) <= 1e-5 * th[0]), np.max(np.abs(lam - th[:k])) / th[0]
    assert abs(info["kyfan"] - th[:k].sum()) <= 1e-5 * th[:k].sum()
    assert np.linalg.norm(S @ S.T - np.eye(k)) <= 1e-5
    G = tucker1.mode1_gram(A.numpy())
    # S carries the Ritz values it reports: tr(S G S^T) = sum theta (oracle G, fp64)
    assert abs(tucker1.kyfan_energy(G, S) - lam.sum()) <= 1e-5 * lam.sum()
    # interlacing with the exact eigenvalues of G
    lam_exact = np.sort(np.linalg.eigvalsh(G))[::-1]
    assert np.all(lam <= lam_exact[:k] * (1 + 1e-6))


@pytest.mark.parametrize("cfg,D,ov,q", [("C1", None, 4, 2), ("C2", 80, 16, 2), ("C3", 20, 16, 3)])
def test_matrix_free_planted_gap_matches_exact_sketch(cfg, D, ov, q):
    """Gap-planted streams (lambda_k / lambda_{k+1} ~ 2): the Krylov sketch reaches the exact
    Tucker1 subspace, on the GPU as in the oracle."""
    c = datagen.planted(cfg, gap=2.0, D_train=D)
    A = datagen.generate(c, "train")
    S, lam, info, st, So, th, K = _run(A, c.k, ov, q)
    S0, lam0, _ = tucker1.tucker1_sketch(A.numpy(), c.k)
    assert tucker1.projector_distance(So, S0) <= 1e-4
    assert tucker1.projector_distance(S, So) <= 1e-4
    np.testing.assert_allclose(lam, lam0[: c.k], rtol=1e-5)


def test_matrix_free_default_start_and_auto_q():
    """No Omega (hash start) and q = auto: q = 2 when (q + 1) p fits min(m, 256)."""
    c = datagen.planted("C2", gap=2.0, D_train=60)
    A = datagen.generate(c, "train")
    S, lam, info, st = tsk.sketch_train_matrix_free(A.cuda(), c.k)
    assert st == 0 and info["block"] == 36 and info["power_iters"] == 2 and info["width"] == 108
    S0, lam0, _ = tucker1.tucker1_sketch(A.numpy(), c.k)
    assert tucker1.projector_distance(S.cpu().double().numpy(), S0) <= 1e-4
    np.testing.assert_allclose(lam.cpu().numpy(), lam0[: c.k], rtol=1e-5)


@pytest.mark.parametrize("subspace", [False, True])
def test_matrix_free_low_rank_breakdown(subspace):
    """Exactly rank-6 stream: G Q_0 has rank 6 < p, so the Krylov block after it breaks down (CholQR
    fails) and is completed with pseudo-random directions (reading mf3); the top-k (k <= 6) sketch
    is still the exact one."""
    c = datagen.lowrank("C2", rank=6).replace(D_train=30)
    A = datagen.generate(c, "train")
    S, lam, info, st = tsk.sketch_train_matrix_free(A.cuda(), 5, oversample=7, power_iters=2, subspace=subspace)
    assert st == 0 and info["repairs"] >= 1
    S0, lam0, _ = tucker1.tucker1_sketch(A.numpy(), 5)
    assert tucker1.projector_distance(S.cpu().double().numpy(), S0) <= 1e-4
    np.testing.assert_allclose(lam.cpu().numpy(), lam0[:5], rtol=1e-5)


def test_matrix_free_ragged_shapes():
    """m not a multiple of 4 or 32, p capped at m, K-tail over the rows: still the oracle's Ritz values."""
    g = torch.Generator().manual_seed(3)
    A = torch.rand(7, 70, 36, generator=g) - 0.3
    S, lam, info, st, So, th, K = _run(A, 6, 10, 2)
    assert info["block"] == 16 and info["width"] == 48
    assert np.all(np.abs(lam - th[:6]) <= 1e-5 * th[0])
    A = torch.rand(3, 10, 8, generator=g)
    S, lam, info, st, So, th, K = _run(A, 3, 20, 0)  # p = m = 10: the full space, exact
    assert info["block"] == 10
    lam0 = np.sort(np.linalg.eigvalsh(tucker1.mode1_gram(A.numpy())))[::-1]
    np.testing.assert_allclose(lam, lam0[:3], rtol=1e-5)


def test_matrix_free_rejects_bad_arguments():
    A = torch.rand(2, 64, 48, device="cuda")
    with pytest.raises(tsk.TskError):
        tsk.sketch_train_matrix_free(A, 10, oversample=200, power_iters=2)   # width > min(m, 256)
    with pytest.raises(tsk.TskError):
        tsk.sketch_train_matrix_free(A, 65)                                   # k > m
    with pytest.raises(tsk.TskError):
        tsk.sketch_train_matrix_free(A[:, :, :46].contiguous(), 4)            # n % 4
    with pytest.raises(tsk.TskError):
        tsk.sketch_train_matrix_free(A[:, :, 1:45].contiguous()[:, :, :44].contiguous().view(-1)[1:1 + 2 * 64 * 40]
                                     .view(2, 64, 40), 4)                     # device A not 16-B aligned


def test_matrix_free_c4_scale():
    """C4 frames (1080 x 1920), 400 training slices: the Krylov sketch (p = 64, q = 2, 5 passes)
    against the exact sketch from the Gram: Ritz values interlace below the exact ones, and the SCW
    test error of the two sketches agrees closely (the metric P:250 is what the sketch is for)."""
    c = datagen.CONFIGS["C4"]
    A = datagen.generate(c, "train", 0, 400, device="cuda")
    T = datagen.generate(c, "test", 0, 16, device="cuda")
    S0, lam0, _, _ = tsk.sketch_train(A, c.k)
    S, lam, info, st = tsk.sketch_train_matrix_free(A, c.k, oversample=4, power_iters=2)
    assert st == 0 and info["width"] == 192 and info["passes"] == 5
    lam0 = lam0.cpu().numpy()
    lam = lam.cpu().numpy()
    # interlacing (exact arithmetic) up to the precision of the compared values: lam0 comes from the 3xTF32
    # Gram, which BASELINE bounds at 1e-5 relative (its truncating split biases it low by ~1e-6, while the
    # Krylov products round to nearest)
    assert np.all(lam <= lam0 * (1 + 1e-5))
    assert lam.sum() >= lam0.sum() * (1 - 1e-2)
    e0 = tsk.scw_error(T, S0, c.r).cpu().numpy()
    e1 = tsk.scw_error(T, S, c.r).cpu().numpy()
    eopt = np.array([oscw.best_rank_r_error(t, c.r) for t in T.cpu().numpy()])
    te0, _ = oscw.test_error(e0, eopt)
    te1, _ = oscw.test_error(e1, eopt)
    assert te1 <= te0 * 1.5 + 1e-3, (te0, te1)


def test_matrix_free_degenerate_sizes():
    """k = 1 and a single training matrix (D = 1): the block Krylov sketch of one frame is the top
    left singular vector of that frame (the oracle, same start block); p = m (q = 0) is exact."""
    g = torch.Generator().manual_seed(11)
    A = torch.rand(1, 40, 24, generator=g)
    S, lam, info, st, So, th, K = _run(A, 1, 3, 3)
    assert st == 0 and info["width"] == 16
    assert abs(lam[0] - th[0]) <= 1e-5 * th[0]
    U, s, _ = np.linalg.svd(A[0].double().numpy())
    assert abs(abs(float(S[0] @ U[:, 0])) - 1.0) <= 1e-6
    np.testing.assert_allclose(lam[0], s[0] ** 2, rtol=1e-5)
    S, lam, info, st, So, th, K = _run(A, 2, 38, 0)   # p = m = 40: exact top-2
    np.testing.assert_allclose(lam, s[:2] ** 2, rtol=1e-5)
