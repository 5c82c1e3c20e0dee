"""End-to-end parity of Algorithm 2 with the float64 oracle: the GPU's own sketch
and errors against the oracle's own sketch and errors on the same seeded streams.

The other parity tests feed the GPU's S into the oracle's SCW (isolating each stage).  Here nothing is
shared: the oracle forms G_o = sum_d A_d A_d^T from the same fp32 frames (in fp64, chunk by chunk at C4),
takes S_o = top-k of G_o, and runs Algorithm 1 with S_o; the GPU runs sketch_train and
scw_error.  BASELINE.json: per-matrix SCW error within 1e-4 relative of the oracle's (1e-6 ||A||_F floor,
reading c13).  The eigengap at k is ~1.0016 at C4 (flat spectrum), so S_gpu and S_o may differ by a
rotation inside the near-degenerate directions at the k boundary; the errors are insensitive to it at the
1e-4 level, which is what this test establishes.  Also checked: Ky Fan energy of S_gpu on
the oracle's G_o, excluding a dominant (frame-mean) pair too (DESIGN reading c15).

Sizes: C1, C2 whole streams; C3 all 400 training / 40 test; C4 all 2000 training frames (oracle Gram in
fp64 ~20-40 s on the host) and 8 sampled test frames.
"""
import numpy as np
import pytest
import torch

import datagen
import paper_2209_14637_b200 as tsk
from oracle import scw as oscw
from oracle import tucker1, tucker2

pytestmark = pytest.mark.gpu


def _oracle_gram_chunked(c, device="cuda", chunk=100):
    """G_o by the oracle's own mode1_gram over chunks of the stream (the definition is a sum over d)."""
    G = np.zeros((c.m, c.m))
    for d0 in range(0, c.D_train, chunk):
        d1 = min(c.D_train, d0 + chunk)
        G += tucker1.mode1_gram(datagen.generate(c, "train", d0, d1, device=device).cpu().numpy())
    return G


@pytest.mark.parametrize("cfg,ntest", [("C1", None), ("C2", None), ("C3", 40), ("C4", 8)])
def test_algorithm2_end_to_end(cfg, ntest):
    c = datagen.CONFIGS[cfg]
    # GPU: the whole training stream -> S
    A = datagen.generate(c, "train", device="cuda")
    S, lam, info, st = tsk.sketch_train(A, c.k)
    assert st == 0
    del A
    torch.cuda.empty_cache()
    # oracle: its own Gram and sketch from the same frames
    G_o = _oracle_gram_chunked(c)
    S_o, lam_o = tucker1.top_k_eigen(G_o, c.k)
    Sd = S.cpu().double().numpy()
    kf = tucker1.kyfan_energy(G_o, Sd)
    tot = lam_o[: c.k].sum()
    assert (tot - kf) <= 1e-6 * tot
    if lam_o[0] >= 20 * lam_o[1]:  # a dominant pair (the frame mean, C3/C4): the rest on its own scale
        assert (tot - kf) <= 1e-6 * lam_o[1: c.k].sum()
    # test stream: GPU errors with S vs oracle errors with S_o
    idx = None
    if ntest is None:
        T = datagen.generate(c, "test", device="cuda")
    else:
        rng = np.random.default_rng(5)
        idx = np.sort(rng.choice(c.D_test, ntest, replace=False))
        T = torch.stack([datagen.generate(c, "test", int(i), int(i) + 1, device="cuda")[0] for i in idx])
    e = tsk.scw_error(T, S, c.r).cpu().numpy()
    Tn = T.cpu().numpy()
    e_o = oscw.scw_errors(Tn, S_o, c.r)
    fro = np.linalg.norm(Tn.reshape(Tn.shape[0], -1).astype(np.float64), axis=1)
    assert np.all(np.abs(e - e_o) <= 1e-4 * e_o + 1e-6 * fro), np.max(np.abs(e - e_o) / e_o)
    # the paper's test-error metric over the sample, GPU vs oracle: mean_b (e_b - eopt_b) / eopt_b
    # moves by at most mean_b |e_b - e_o,b| / eopt_b, so the per-matrix bound above (1e-4 e_o + 1e-6 ||A||,
    # BASELINE.json) bounds it -- the metric is a difference of nearly equal errors (~1e-4 at C1), so a
    # relative tolerance on it would ask ~1e-7 of each error, which BASELINE does not
    eopt = np.array([oscw.best_rank_r_error(a, c.r) for a in Tn])
    bound = np.mean((1e-4 * e_o + 1e-6 * fro) / eopt)
    assert abs(oscw.test_error(e, eopt)[0] - oscw.test_error(e_o, eopt)[0]) <= bound


@pytest.mark.parametrize("cfg,nsample", [("C3", 6), ("C4", 4)])
def test_scw_factors_multitile(cfg, nsample):
    """sketch_apply_scw's factors L, R, sigma at multi-tile sizes (m, n >= 768) against the oracle's
    Algorithm 1 factors: A_hat = L R^T, sigma = singular values of AV, R orthonormal."""
    c = datagen.CONFIGS[cfg]
    rng = np.random.default_rng(7)
    q, _ = np.linalg.qr(rng.standard_normal((c.m, c.k)))
    S = torch.tensor(q.T.copy(), dtype=torch.float32)
    T = datagen.generate(c, "test", 0, nsample)
    L, R, sig = tsk.sketch_apply_scw(T.cuda(), S.cuda(), c.r)
    L, R, sig = L.double().cpu().numpy(), R.double().cpu().numpy(), sig.double().cpu().numpy()
    for b in range(nsample):
        Lo, so, Ro = oscw.scw_factors(T[b].numpy(), S.double().numpy(), c.r)
        Ah, Ah_o = L[b] @ R[b].T, Lo @ Ro.T
        assert np.linalg.norm(Ah - Ah_o) / np.linalg.norm(Ah_o) <= 1e-5
        np.testing.assert_allclose(sig[b], so, rtol=1e-5)
        assert np.linalg.norm(R[b].T @ R[b] - np.eye(c.r)) <= 1e-5
        # L = U_r diag(sigma): its column norms are the singular values
        np.testing.assert_allclose(np.linalg.norm(L[b], axis=0), so, rtol=1e-5)


@pytest.mark.filterwarnings("ignore:sketch_train_two_sided")
@pytest.mark.parametrize("cfg,k,l,D,ntest", [("C1", 10, 8, None, None), ("C2", 20, 20, 60, 20),
                                             ("C3", 40, 40, 12, 6)])
def test_two_sided_end_to_end(cfg, k, l, D, ntest):
    """Algorithm 4 end to end: the GPU's HOOI factors (S, W) and two-sided errors against
    the oracle HOOI's (S_o, W_o) and its errors, on the same frames (same HOSVD start and sweep count)."""
    c = datagen.CONFIGS[cfg]
    A = datagen.generate(c, "train", 0, D or c.D_train)
    S, W, info, st = tsk.sketch_train_two_sided(A.cuda(), k, l, max_sweeps=4, rel_tol=1e-14)
    So, Wo, _, _ = tucker2.hooi_tucker2(A.numpy().astype(np.float64), k, l, max_iters=4, rel_tol=1e-14)
    T = datagen.generate(c, "test", 0, ntest)
    r = min(c.r, k, l)
    e = tsk.two_sided_scw_error(T.cuda(), S, W, r).cpu().numpy()
    e_o = tucker2.two_sided_scw_errors(T.numpy(), So, Wo, r)
    fro = np.linalg.norm(T.numpy().reshape(T.shape[0], -1).astype(np.float64), axis=1)
    assert np.all(np.abs(e - e_o) <= 1e-4 * e_o + 1e-6 * fro), np.max(np.abs(e - e_o) / e_o)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4"])
def test_scw_error_formulas_agree(cfg):
    """scw_error's Pythagorean error (mode 0, reading c17) against its dense residual (mode 1) on the same
    stream and sketch: both are Algorithm 1's ||A - [AV]_r V^T||_F, so they agree within the
    per-matrix BASELINE tolerance; the dense residual also takes over below tau ||A||^2 (forced here with
    tau = 0.999: every matrix then goes through the fallback, which must equal mode 1 bit for bit)."""
    c = datagen.CONFIGS[cfg]
    T = datagen.generate(c, "test", 0, min(c.D_test, 64), device="cuda")
    q, _ = np.linalg.qr(np.random.default_rng(3).standard_normal((c.m, c.k)))
    S = torch.tensor(q.T.copy(), dtype=torch.float32, device="cuda")
    try:
        tsk.set_scw_error_mode(1)
        e_d = tsk.scw_error(T, S, c.r).cpu().numpy()
        tsk.set_scw_error_mode(0, 0.999)
        e_f = tsk.scw_error(T, S, c.r).cpu().numpy()
        tsk.set_scw_error_mode(0)
        e_p = tsk.scw_error(T, S, c.r).cpu().numpy()
    finally:
        tsk.set_scw_error_mode(0)
    fro = np.linalg.norm(T.cpu().numpy().reshape(T.shape[0], -1).astype(np.float64), axis=1)
    assert np.all(np.abs(e_p - e_d) <= 1e-4 * e_d + 1e-6 * fro), np.max(np.abs(e_p - e_d) / e_d)
    np.testing.assert_array_equal(e_f, e_d)
