"""Seeded random shapes through every entry point against the float64 oracle (the fixed-seed core of
scripts/random_sweep*.py, which found the m % 4 != 0 SCW rejection and the two-sided workspace
under-allocation).  Tolerances as the parity tests: Gram rel-F <= 1e-5; SCW errors within 1e-4 relative
+ 1e-6 ||A||_F (reading c13); Ky Fan deficit <= 1e-6; matrix-free Ritz values within 1e-5 theta_1."""
import numpy as np
import pytest
import torch

import datagen
import paper_2209_14637_b200 as tsk
from oracle import matrix_free as omf
from oracle import scw as oscw
from oracle import tucker1, tucker2

pytestmark = pytest.mark.gpu


def _orth_rows(rng, k, m):
    q, _ = np.linalg.qr(rng.standard_normal((m, k)))
    return torch.tensor(q.T.copy(), dtype=torch.float32)


def _errs_close(e, eo, T):
    fro = np.linalg.norm(T.numpy().reshape(T.shape[0], -1).astype(np.float64), axis=1)
    return np.all(np.abs(e - eo) <= 1e-4 * eo + 1e-6 * fro)


@pytest.mark.parametrize("seed", range(6))
def test_random_one_sided_path(seed):
    rng = np.random.default_rng(1000 + seed)
    m = int(rng.integers(2, 700)); n = int(rng.integers(1, 200)) * 4; D = int(rng.integers(1, 12))
    A = torch.from_numpy(rng.random((D, m, n), dtype=np.float32) - 0.3)
    G, _ = tsk.sketch_gram(A.cuda())
    Go = tucker1.mode1_gram(A.numpy())
    assert np.linalg.norm(G.cpu().numpy() - Go) / np.linalg.norm(Go) <= 1e-5
    k = int(rng.integers(1, min(m, 60) + 1)); r = int(rng.integers(1, min(k, n, m) + 1))
    S, lam, info, st = tsk.sketch_topk(G, k)
    w = np.sort(np.linalg.eigvalsh(Go))[::-1]
    assert (w[:k].sum() - tucker1.kyfan_energy(Go, S.cpu().double().numpy())) <= 1e-6 * w[:k].sum()
    T = torch.from_numpy(rng.random((3, m, n), dtype=np.float32) - 0.3)
    e = tsk.scw_error(T.cuda(), S, r).cpu().numpy()
    assert _errs_close(e, oscw.scw_errors(T.numpy(), S.cpu().double().numpy(), r), T)


@pytest.mark.parametrize("seed", range(4))
def test_random_two_sided_and_matrix_free(seed):
    rng = np.random.default_rng(2000 + seed)
    m = int(rng.integers(1, 100)) * 4; n = int(rng.integers(1, 100)) * 4; D = int(rng.integers(1, 10))
    A = torch.from_numpy(rng.random((D, m, n), dtype=np.float32) - 0.3)
    T = torch.from_numpy(rng.random((3, m, n), dtype=np.float32) - 0.3)
    G2 = tsk.sketch_gram_mode2(A.cuda()).cpu().numpy()
    G2o = tucker2.mode2_gram(A.numpy())
    assert np.linalg.norm(G2 - G2o) / np.linalg.norm(G2o) <= 1e-5
    k = int(rng.integers(1, min(m, 40) + 1)); l = int(rng.integers(1, min(n, 40) + 1))
    r = int(rng.integers(1, min(k, l) + 1))
    S, W = _orth_rows(rng, k, m), _orth_rows(rng, l, n)
    e2 = tsk.two_sided_scw_error(T.cuda(), S.cuda(), W.cuda(), r).cpu().numpy()
    assert _errs_close(e2, tucker2.two_sided_scw_errors(T.numpy(), S.double().numpy(), W.double().numpy(), r), T)
    kk = int(rng.integers(1, min(m, 30) + 1)); ov = int(rng.integers(1, 20))
    p = min((kk + ov + 3) // 4 * 4, m)
    q = int(rng.integers(0, 3))
    if (q + 1) * p <= min(m, 256):
        om = datagen.start_block(m, p, seed)
        Sm, lamm, info, st = tsk.sketch_train_matrix_free(A.cuda(), kk, oversample=ov, power_iters=q, omega=om.cuda())
        So, th, K = omf.matrix_free_sketch(A.numpy(), kk, om.numpy(), q)
        assert np.max(np.abs(lamm.cpu().numpy() - th[:kk])) <= 1e-5 * th[0]


@pytest.mark.parametrize("kind", ["dominant", "clustered", "rankdef", "steep", "dominant2"])
def test_eigensolver_spectra(kind):
    """Synthetic spectra for the subspace-iteration eigensolver (m > 256): a dominant eigenvalue above a
    flat rest (the case the residual-only stopping rule under-converged), clusters, rank deficiency, and a
    steep power-law top over a nearly flat bulk below a dominant mean (the C4 shape, exaggerated: the
    filter runs at the 1e13 steep-spectrum range)."""
    rng = np.random.default_rng({"dominant": 1, "clustered": 2, "rankdef": 3, "steep": 4, "dominant2": 5}[kind])
    m, k = 700, 40
    if kind == "dominant":
        lam = 1.0 + rng.random(m)
        lam[0] = 1e5
    elif kind == "dominant2":  # a dominant pair only 50x above the next, locked by the power pre-pass with a
        lam = 1.0 + 0.05 * rng.random(m)  # residual above 0.1 tol theta_k (its error lies along the top pair)
        lam[1] = 2e4
        lam[0] = 1e6
    elif kind == "steep":
        lam = 1.0 + 0.05 * rng.random(m)
        lam[1:13] += 2000.0 * np.arange(1, 13) ** -1.5
        lam[0] = 1e6
    elif kind == "clustered":
        lam = np.repeat(rng.random(m // 8 + 1) * 10, 8)[:m]
    else:
        lam = np.zeros(m)
        lam[:25] = rng.random(25) + 0.1
    U, _ = np.linalg.qr(rng.standard_normal((m, m)))
    G = (U * lam) @ U.T
    G = 0.5 * (G + G.T)
    S, l, info, st = tsk.sketch_topk(torch.tensor(G, device="cuda"), k)
    Sd = S.cpu().double().numpy()
    w = np.sort(lam)[::-1]
    assert (w[:k].sum() - tucker1.kyfan_energy(G, Sd)) <= 1e-6 * w[:k].sum()
    assert np.linalg.norm(Sd @ Sd.T - np.eye(k)) <= 1e-5
    if kind in ("steep", "dominant2"):
        # converged without a fallback status; Ritz values below their eigenvalues (interlacing) and within
        # the Ky Fan stopping deficit of them (reading c15); the bulk gap at k is ~1.0 -- no projector claim
        assert st == 0, info.as_dict()
        short = w[:k] - l.cpu().numpy()
        assert np.all(short >= -1e-12 * w[0]) and short.sum() <= 1e-6 * w[:k].sum() + 1e-12 * w[0]
