"""The whole hot path at BASELINE.json's full C4 size, in the launch configuration bench.py times
(D_train = 2000 training frames, 500 test frames, one sketch_train + one scw_error call).

The oracle cannot redo the fp64 Gram of 2000 frames in seconds, so the check is split where the
oracle can follow (③: sampled outputs / properties that hold at any size):
- G: sampled rows of the GPU Gram against the oracle's entry formula (as test_gram_full_size_sampled);
- S: against numpy's eigh of the GPU's G in fp64 -- Ky Fan energy and the Ritz backward error of every
  row of S (the eigensolver's stopping rule, reading c15), orthonormal rows, sign rule c5;
- SCW: the errors of a sample of the 500 test matrices against the oracle's Algorithm 1 with the
  GPU's S (1e-4 relative + 1e-6 ||A||_F, reading c13), all 500 above the Eckart-Young optimum of
  their own sample.
"""
import numpy as np
import pytest
import torch

import datagen
import paper_2209_14637_b200 as tsk
from oracle import scw as oscw
from oracle import tucker1

pytestmark = pytest.mark.gpu


def test_c4_full_size_path():
    c = datagen.CONFIGS["C4"]
    A = datagen.generate(c, "train", device="cuda")
    T = datagen.generate(c, "test", device="cuda")
    assert A.shape[0] == 2000 and T.shape[0] == 500
    G = torch.empty(c.m, c.m, dtype=torch.float64, device="cuda")
    S, lam, info, st = tsk.sketch_train(A, c.k, G64_out=G)
    err = tsk.scw_error(T, S, c.r).cpu().numpy()
    assert st == 0 and err.shape == (500,) and np.all(np.isfinite(err))

    # G: sampled entries, one by one from the fp32 frames in fp64
    rng = np.random.default_rng(3)
    R = np.unique(np.concatenate([rng.choice(c.m, 14, replace=False), [0, c.m - 1]]))
    Ar = A[:, torch.tensor(R, device="cuda"), :].double().cpu().numpy()
    Go = np.einsum("dik,djk->ij", Ar, Ar)
    Gg = G.cpu().numpy()
    assert np.max(np.abs(Gg[np.ix_(R, R)] - Go) / np.abs(Go)) <= 1e-5
    del A, Ar

    # S against the eigendecomposition of the (sampled-validated) G in fp64
    w, U = np.linalg.eigh(Gg)
    w, U = w[::-1], U[:, ::-1]
    Sd = S.cpu().double().numpy()
    lamg = lam.cpu().numpy()
    assert np.linalg.norm(Sd @ Sd.T - np.eye(c.k)) <= 1e-5
    assert abs(tucker1.kyfan_energy(Gg, Sd) - w[: c.k].sum()) <= 1e-6 * w[: c.k].sum()
    # the k - 1 directions below the dominant frame mean on their own scale (DESIGN reading c15: the
    # stopping rule measures residuals against theta_k, not theta_1)
    assert w[0] >= 20 * w[1]
    assert abs(tucker1.kyfan_energy(Gg, Sd) - w[: c.k].sum()) <= 1e-6 * w[1: c.k].sum()
    # Ritz values (fp64 products) relative to the k-th eigenvalue, not the dominant one
    assert np.max(np.abs(lamg - w[: c.k])) <= 1e-6 * w[c.k - 1]
    res = np.linalg.norm(Gg @ Sd.T - Sd.T * (np.einsum("ij,jk,ik->i", Sd, Gg, Sd))[None, :], axis=0)
    assert np.max(res) <= 1e-5 * w[0]
    big = np.argmax(np.abs(Sd), axis=1)
    assert np.all(Sd[np.arange(c.k), big] > 0)

    # SCW: sampled test matrices against the oracle's Algorithm 1 with the GPU's S
    pick = np.unique(np.concatenate([rng.choice(500, 5, replace=False), [0, 499]]))
    Tp = T[torch.tensor(pick, device="cuda")].cpu().numpy()
    eo = oscw.scw_errors(Tp, Sd, c.r)
    fro = np.linalg.norm(Tp.reshape(len(pick), -1).astype(np.float64), axis=1)
    assert np.all(np.abs(err[pick] - eo) <= 1e-4 * eo + 1e-6 * fro), (err[pick], eo)
    eopt = np.array([oscw.best_rank_r_error(a, c.r) for a in Tp])
    assert np.all(err[pick] >= eopt * (1 - 1e-6))
