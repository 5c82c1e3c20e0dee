"""BASELINE.json configs[4] (C5: m = n = 4096, k = 100, r = 50) on the GPU against the float64 oracle.

The full C5 training stream is 2000 x 64 MB; the oracle's Gram of it takes ~20 min on the host, so
parity is checked (i) on a reduced stream D_train = 24 (same generator, shapes, k, r) through the
whole path -- Gram rel-F, sketch Ky Fan deficit / orthonormality, SCW errors -- (ii) at the full
C5 matrix shape with D = 64 on sampled Gram entries computed one by one in fp64, and (iii) on the full
2000-frame stream through sampled Gram entries and properties of the sketch that hold at any size.  The two-sided
entry points are exercised at C5's m, n with k = l = 100."""
import numpy as np
import pytest
import torch

import datagen
import paper_2209_14637_b200 as tsk
from oracle import scw as oscw
from oracle import tucker1, tucker2

pytestmark = pytest.mark.gpu

C5 = datagen.CONFIGS["C5"]


@pytest.fixture(scope="module")
def c5_small():
    A = datagen.generate(C5, "train", 0, 24, device="cuda")
    T = datagen.generate(C5, "test", 0, 3, device="cuda")
    return A, T


def test_c5_gram_sketch_scw(c5_small):
    A, T = c5_small
    G = torch.empty(C5.m, C5.m, dtype=torch.float64, device="cuda")
    S, lam, info, st = tsk.sketch_train(A, C5.k, G64_out=G)
    An = A.cpu().numpy()
    Go = tucker1.mode1_gram(An)
    assert float(np.linalg.norm(G.cpu().numpy() - Go) / np.linalg.norm(Go)) <= 1e-5
    lam_o = np.linalg.eigvalsh(Go)[::-1]
    Sg = S.cpu().double().numpy()
    deficit = (lam_o[:C5.k].sum() - tucker1.kyfan_energy(Go, Sg)) / lam_o[:C5.k].sum()
    assert abs(deficit) <= 1e-6
    assert np.linalg.norm(Sg @ Sg.T - np.eye(C5.k)) <= 1e-5
    err = tsk.scw_error(T, S, C5.r).cpu().numpy()
    eo = oscw.scw_errors(T.cpu().numpy(), Sg, C5.r)
    fro = np.linalg.norm(T.cpu().double().numpy().reshape(T.shape[0], -1), axis=1)
    assert np.all(np.abs(err - eo) <= 1e-4 * eo + 1e-6 * fro)


def test_c5_gram_full_shape_sampled():
    A = datagen.generate(C5, "train", 0, 64, device="cuda")
    G, info = tsk.sketch_gram(A)
    rng = np.random.default_rng(2)
    R = np.unique(np.concatenate([rng.choice(C5.m, 22, replace=False), [0, C5.m - 1]]))
    Ar = A[:, torch.tensor(R, device="cuda"), :].double().cpu().numpy()
    Go = np.einsum("dik,djk->ij", Ar, Ar)
    Gg = G.cpu().numpy()[np.ix_(R, R)]
    # zero-mean data: off-diagonal entries may be small; relative to the diagonal scale
    scale = np.sqrt(np.outer(np.diag(Go), np.diag(Go)))
    assert np.max(np.abs(Gg - Go) / scale) <= 1e-5


def test_c5_two_sided_scw(c5_small):
    A, T = c5_small
    S = torch.tensor(np.linalg.qr(np.random.default_rng(1).standard_normal((C5.m, C5.k)))[0].T.copy(),
                     dtype=torch.float32, device="cuda")
    W = torch.tensor(np.linalg.qr(np.random.default_rng(2).standard_normal((C5.n, C5.k)))[0].T.copy(),
                     dtype=torch.float32, device="cuda")
    err = tsk.two_sided_scw_error(T, S, W, C5.r).cpu().numpy()
    eo = tucker2.two_sided_scw_errors(T.cpu().numpy(), S.cpu().double().numpy(), W.cpu().double().numpy(), C5.r)
    fro = np.linalg.norm(T.cpu().double().numpy().reshape(T.shape[0], -1), axis=1)
    assert np.all(np.abs(err - eo) <= 1e-4 * eo + 1e-6 * fro)


def test_c5_full_stream_properties():
    """C5 at its full size (D_train = 2000 frames of 4096 x 4096, generated and accumulated in chunks of 100
    as the streaming use does): sampled Gram entries in fp64 from the same frames (one by one, the definition), then the
    sketch through properties that hold at any size -- Ky Fan deficit against fp64 eigvalsh of the
    accumulated G, orthonormal rows -- and SCW errors of sampled test matrices against the oracle."""
    D, ch = C5.D_train, 100
    G = torch.zeros(C5.m, C5.m, dtype=torch.float64, device="cuda")
    rng = np.random.default_rng(4)
    R = np.unique(np.concatenate([rng.choice(C5.m, 14, replace=False), [0, C5.m - 1]]))
    Rt = torch.tensor(R, device="cuda")
    Go = np.zeros((len(R), len(R)))
    for d0 in range(0, D, ch):
        A = datagen.generate(C5, "train", d0, d0 + ch, device="cuda")
        tsk.sketch_gram(A, G64=G, accumulate=d0 > 0)
        Ar = A[:, Rt, :].double().cpu().numpy()
        Go += np.einsum("dik,djk->ij", Ar, Ar)
        del A
    Gg = G[Rt][:, Rt].cpu().numpy()
    scale = np.sqrt(np.outer(np.diag(Go), np.diag(Go)))
    assert np.max(np.abs(Gg - Go) / scale) <= 1e-5
    S, lam, info, st = tsk.sketch_topk(G, C5.k)
    assert st == 0
    Sd = S.double()
    lam_ref = torch.linalg.eigvalsh(G).flip(0)[: C5.k].sum().item()
    kf = torch.trace(Sd @ G @ Sd.T).item()
    assert abs(lam_ref - kf) <= 1e-6 * lam_ref
    assert torch.linalg.norm(Sd @ Sd.T - torch.eye(C5.k, device="cuda", dtype=torch.float64)).item() <= 1e-5
    T = torch.stack([datagen.generate(C5, "test", i, i + 1, device="cuda")[0] for i in (0, 100, 255)])
    err = tsk.scw_error(T, S, C5.r).cpu().numpy()
    eo = oscw.scw_errors(T.cpu().numpy(), S.cpu().double().numpy(), C5.r)
    fro = np.linalg.norm(T.cpu().double().numpy().reshape(T.shape[0], -1), axis=1)
    assert np.all(np.abs(err - eo) <= 1e-4 * eo + 1e-6 * fro)
