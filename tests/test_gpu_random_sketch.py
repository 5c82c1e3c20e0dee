"""Random-sketch baselines through the same GPU SCW kernels.

The untrained sketches (CountSketch signs, Gaussian N(0, 1/k); datagen) are not row-orthonormal;
Algorithm 1 only uses rowspace(S A), which the GPU computes (pivoted-Cholesky basis)
rather than assumes.  Parity: per-matrix errors within 1e-4 of the float64 oracle's SCW with the same
S.  Pattern (P:27, P:266 in spirit; SPEC acceptance 6): on the synthetic streams the trained
(Tucker1) sketch's test error (metric P:250) is below both random sketches'.
"""
import numpy as np
import pytest
import torch

import datagen
import paper_2209_14637_b200 as tsk
from oracle import scw as oscw

pytestmark = pytest.mark.gpu


def _errs(T, S, r):
    err = tsk.scw_error(T.cuda(), S.cuda(), r).cpu().numpy()
    eo = oscw.scw_errors(T.numpy(), S.double().numpy(), r)
    fro = np.linalg.norm(T.numpy().reshape(T.shape[0], -1).astype(np.float64), axis=1)
    assert np.all(np.abs(err - eo) <= 1e-4 * eo + 1e-6 * fro)
    return err


@pytest.mark.parametrize("cfg,ntest", [("C1", None), ("C2", 12), ("C3", 4)])
def test_random_sketch_scw_parity(cfg, ntest):
    c = datagen.CONFIGS[cfg]
    T = datagen.generate(c, "test", 0, ntest)
    _errs(T, datagen.random_sign_sketch(c.k, c.m, seed=1), c.r)
    _errs(T, datagen.random_gaussian_sketch(c.k, c.m, seed=2), c.r)


@pytest.mark.parametrize("cfg,ntrain,ntest", [("C1", None, None), ("C2", 100, 40)])
def test_trained_sketch_beats_random(cfg, ntrain, ntest):
    c = datagen.CONFIGS[cfg]
    A = datagen.generate(c, "train", 0, ntrain)
    T = datagen.generate(c, "test", 0, ntest)
    S, lam, info, st = tsk.sketch_train(A.cuda(), c.k)
    eopt = np.array([oscw.best_rank_r_error(t, c.r) for t in T.numpy()])
    te = {}
    for name, Sk in [("tensor", S.cpu()), ("sign", datagen.random_sign_sketch(c.k, c.m, seed=5)),
                     ("gauss", datagen.random_gaussian_sketch(c.k, c.m, seed=6))]:
        e = tsk.scw_error(T.cuda(), Sk.cuda(), c.r).cpu().numpy()
        te[name], _ = oscw.test_error(e, eopt)
    assert te["tensor"] < te["sign"] and te["tensor"] < te["gauss"], te
