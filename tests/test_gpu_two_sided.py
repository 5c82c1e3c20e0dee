"""Parity of the two-sided variant on the GPU with the float64 oracle
(oracle/tucker2.py): the mode-2 Gram, Tucker2 by HOOI (Eq. (9), Algorithm 5) and two-sided SCW
(Algorithm 3), through the C ABI.

Tolerances: Gram relative Frobenius error <= 1e-5 (as the mode-1 Gram); SCW errors within 1e-4
relative (+ 1e-6 ||A||_F floor, reading c13); the direct fp64 residual of the GPU's HOOI factors
within 1e-6 relative of the oracle HOOI's (same HOSVD init and updates; the residual is stationary
at the optimum, so S/W rounding enters quadratically); the GPU's residual bookkeeping (from 3xTF32
projected Grams) within 1e-4 sweep by sweep; projector distances <= 1e-4 only on gap-planted data
(reading c16).
"""
import numpy as np
import pytest
import torch

import datagen
import paper_2209_14637_b200 as tsk
from oracle import scw as oscw
from oracle import tucker1, tucker2

pytestmark = pytest.mark.gpu


def relF(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def rand_stack(D, m, n, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.rand(D, m, n, generator=g) - 0.25


def orth_rows(k, m, seed):
    q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((m, k)))
    return torch.tensor(q.T.copy(), dtype=torch.float32)


@pytest.mark.parametrize("D,m,n", [(3, 64, 48), (5, 132, 40), (4, 256, 256), (2, 100, 300), (3, 1080, 1920),
                                   (1, 8, 4), (6, 36, 260)])
def test_gram_mode2_matches_oracle(D, m, n):
    A = rand_stack(D, m, n, seed=D * 100 + n)
    G = tsk.sketch_gram_mode2(A.cuda()).cpu().numpy()
    Go = tucker2.mode2_gram(A.numpy())
    assert relF(G, Go) <= 1e-5
    np.testing.assert_array_equal(G, G.T)


def test_gram_mode2_accumulate():
    A = rand_stack(6, 64, 96, seed=3)
    G = tsk.sketch_gram_mode2(A[:4].cuda())
    tsk.sketch_gram_mode2(A[4:].cuda(), G64=G, accumulate=True)
    assert relF(G.cpu().numpy(), tucker2.mode2_gram(A.numpy())) <= 1e-5


@pytest.mark.parametrize("cfg,k,l,D", [("C1", 10, 8, None), ("C2", 20, 20, 60), ("C3", 40, 40, 12)])
def test_hooi_matches_oracle(cfg, k, l, D):
    c = datagen.CONFIGS[cfg]
    A = datagen.generate(c, "train", 0, D or c.D_train)
    S, W, info, st = tsk.sketch_train_two_sided(A.cuda(), k, l, max_sweeps=4, rel_tol=1e-14)
    S, W = S.cpu().double().numpy(), W.cpu().double().numpy()
    Ad = A.numpy().astype(np.float64)
    So, Wo, hist_o, _ = tucker2.hooi_tucker2(Ad, k, l, max_iters=4, rel_tol=1e-14)
    hist = info["residual_history"]
    assert info["sweeps"] == len(hist_o) - 1
    # quality of the GPU's factors: their direct fp64 residual equals the oracle HOOI's (the residual
    # is stationary at the optimum, so factor rounding enters quadratically)
    res_direct = tucker2.tucker2_residual(Ad, S, W)
    assert res_direct == pytest.approx(hist_o[-1], rel=1e-6)
    # the GPU's own bookkeeping ||A||^2 - (top-l energy of the 3xTF32 projected Gram) tracks the oracle
    # sweep by sweep; its ~1e-6 relative energy error is amplified by ||A||^2 / residual^2
    np.testing.assert_allclose(hist, hist_o[:len(hist)], rtol=1e-4)
    assert res_direct == pytest.approx(hist[-1], rel=1e-4)
    assert all(b <= a * (1 + 1e-7) for a, b in zip(hist, hist[1:]))   # monotone
    np.testing.assert_allclose(S @ S.T, np.eye(k), atol=1e-5)
    np.testing.assert_allclose(W @ W.T, np.eye(l), atol=1e-5)
    assert info["a_fro2"] == pytest.approx(float(np.sum(Ad * Ad)), rel=1e-5)  # trace of the 3xTF32 Gram


def test_hooi_planted_projectors():
    """Exact multilinear rank (k, l) plus small noise: S and W are pinned by large gaps."""
    rng = np.random.default_rng(7)
    D, m, n, k, l = 16, 128, 96, 8, 12
    U0 = np.linalg.qr(rng.standard_normal((m, k)))[0]
    V0 = np.linalg.qr(rng.standard_normal((n, l)))[0]
    A = np.stack([U0 @ rng.standard_normal((k, l)) @ V0.T + 1e-3 * rng.standard_normal((m, n))
                  for _ in range(D)]).astype(np.float32)
    S, W, info, st = tsk.sketch_train_two_sided(torch.tensor(A).cuda(), k, l, max_sweeps=5)
    So, Wo, hist_o, _ = tucker2.hooi_tucker2(A.astype(np.float64), k, l, max_iters=5)
    assert tucker1.projector_distance(S.cpu().double().numpy(), So) <= 1e-4
    assert tucker1.projector_distance(W.cpu().double().numpy(), Wo) <= 1e-4


def _scw2_parity(T, S, W, r):
    err = tsk.two_sided_scw_error(T.cuda(), S.cuda(), W.cuda(), r).cpu().numpy()
    eo = tucker2.two_sided_scw_errors(T.numpy(), S.double().numpy(), W.double().numpy(), r)
    fro = np.linalg.norm(T.numpy().reshape(T.shape[0], -1).astype(np.float64), axis=1)
    assert np.all(np.abs(err - eo) <= 1e-4 * eo + 1e-6 * fro), np.max(np.abs(err - eo) / eo)
    return err, eo


@pytest.mark.parametrize("cfg,k,l,ntest", [("C1", 12, 8, None), ("C2", 20, 20, 16), ("C3", 40, 40, 6),
                                           ("C4", 60, 60, 3)])
def test_two_sided_scw_matches_oracle(cfg, k, l, ntest):
    c = datagen.CONFIGS[cfg]
    T = datagen.generate(c, "test", 0, ntest)
    S, W = orth_rows(k, c.m, 1), orth_rows(l, c.n, 2)
    _scw2_parity(T, S, W, c.r if c.r <= min(k, l) else min(k, l))


def test_two_sided_scw_with_trained_pair():
    c = datagen.CONFIGS["C2"]
    A = datagen.generate(c, "train", 0, 40)
    T = datagen.generate(c, "test", 0, 8)
    S, W, info, st = tsk.sketch_train_two_sided(A.cuda(), 20, 20, max_sweeps=3)
    err, eo = _scw2_parity(T, S.cpu(), W.cpu(), c.r)
    # the one-sided SCW with the same S is never worse (row space of the two-sided A_hat lies in
    # rowspace(S A), where SCW is the best rank-r approximation)
    e1 = tsk.scw_error(T.cuda(), S, c.r).cpu().numpy()
    assert np.all(e1 <= err * (1 + 1e-5))


def test_two_sided_scw_special_cases():
    rng = np.random.default_rng(5)
    m, n, r = 64, 48, 5
    T = torch.tensor(rng.standard_normal((3, m, n)), dtype=torch.float32)
    # full factors S = I_m, W = I_n: A_hat = [A]_r (Eckart-Young)
    e = tsk.two_sided_scw_error(T.cuda(), torch.eye(m).cuda(), torch.eye(n).cuda(), r).cpu().numpy()
    eo = np.array([oscw.best_rank_r_error(a, r) for a in T.numpy()])
    np.testing.assert_allclose(e, eo, rtol=1e-5)
    # W = I_n: identical to the one-sided SCW
    S = orth_rows(10, m, 9)
    e2 = tsk.two_sided_scw_error(T.cuda(), S.cuda(), torch.eye(n).cuda(), r).cpu().numpy()
    e1 = tsk.scw_error(T.cuda(), S.cuda(), r).cpu().numpy()
    np.testing.assert_allclose(e2, e1, rtol=1e-5)
    # exactly rank 3 <= r: zero error
    L0 = rng.standard_normal((3, m, 3)) @ rng.standard_normal((3, 3, n))
    Tl = torch.tensor(L0, dtype=torch.float32)
    e3 = tsk.two_sided_scw_error(Tl.cuda(), orth_rows(8, m, 1).cuda(), orth_rows(8, n, 2).cuda(), 3).cpu().numpy()
    assert np.all(e3 <= 1e-5 * np.linalg.norm(L0.reshape(3, -1), axis=1))
    # factors: L R^T equals the oracle's A_hat
    L, R, sig = tsk.sketch_apply_two_sided_scw(T[:1].cuda(), S.cuda(), orth_rows(12, n, 4).cuda(), r)
    Ah = (L[0].double() @ R[0].double().T).cpu().numpy()
    Aho = tucker2.two_sided_scw(T[0].numpy(), S.double().numpy(), orth_rows(12, n, 4).double().numpy(), r)
    assert relF(Ah, Aho) <= 1e-5


@pytest.mark.parametrize("m,n,k,l,r", [(188, 204, 18, 6, 5), (96, 40, 30, 4, 3)])
def test_two_sided_scw_k_much_larger_than_l_fresh_context(m, n, k, l, r):
    """k >> l on a FRESH context (workspaces sized by this call alone): the small-matrix workspace of the
    two-sided SCW used to be short by k(k - l) - l doubles per matrix, corrupting the later matrices of
    a batch (found by scripts/random_sweep2.py)."""
    rng = np.random.default_rng(m + k)
    T = torch.from_numpy(rng.random((3, m, n), dtype=np.float32) - 0.3)
    S = torch.tensor(orth_rows(k, m, 1).numpy())
    W = torch.tensor(orth_rows(l, n, 2).numpy())
    ctx = tsk.Context(0)
    e = tsk.two_sided_scw_error(T.cuda(), S.cuda(), W.cuda(), r, ctx=ctx).cpu().numpy()
    ctx.close()
    eo = tucker2.two_sided_scw_errors(T.numpy(), S.double().numpy(), W.double().numpy(), r)
    assert np.all(np.abs(e - eo) <= 1e-4 * eo), (e, eo)
