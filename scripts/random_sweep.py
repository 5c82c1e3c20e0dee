"""Randomised robustness sweeps of every entry point against the float64 oracle (developer check; the
fixed-seed core runs in tests/test_gpu_random_shapes.py).  One script, six suites:
  core     random shapes: Gram, sketch (Ky Fan), SCW errors          (--big: m in [257, 1500], k <= 100)
  f_rows   mode-2 Gram, HOOI + two-sided SCW, matrix-free sketch, SCW factors
  api      host vs device pointers (bitwise), streamed accumulate, G32 output, factors vs errors
  mixed    HOOI vs the oracle HOOI, warm-started top-k, split-K Grams with thousands of thin slices
  spectra  the eigensolver on synthetic spectra (flat, geometric, clustered, rank-deficient, dominant, two-gap)
  limits   SCW with k in [90, 128], r up to 64; two-sided SCW with k, l up to 116
Found so far: SCW rejecting m % 4 != 0 (core), the two-sided workspace under-allocation (f_rows), a dominant
eigenvalue stopping the round-1 eigensolver early (spectra).
  python scripts/random_sweep.py SUITE [n_cases] [seed] [--big]"""
import os, sys, time, warnings
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402
from oracle import matrix_free as omf, scw as oscw, tucker1, tucker2  # noqa: E402


def orth_rows(rng, k, m):
    q, _ = np.linalg.qr(rng.standard_normal((m, k)))
    return torch.tensor(q.T.copy(), dtype=torch.float32)


def suite_core(ncase, rng):
    bad = 0
    big = "--big" in sys.argv
    for t in range(ncase):
        m = int(rng.integers(257, 1500)) if big else int(rng.integers(2, 700))
        n = int(rng.integers(1, 200)) * 4; D = int(rng.integers(1, 12))
        A = torch.from_numpy(rng.random((D, m, n), dtype=np.float32) - 0.3)
        G, _ = tsk.sketch_gram(A.cuda())
        Go = tucker1.mode1_gram(A.numpy())
        ge = float(np.linalg.norm(G.cpu().numpy() - Go) / np.linalg.norm(Go))
        k = int(rng.integers(1, min(m, 100 if big else 60) + 1)); r = int(rng.integers(1, min(k, n, m, 64) + 1))
        S, lam, info, st = tsk.sketch_topk(G, k)
        Sd = S.cpu().double().numpy()
        w = np.sort(np.linalg.eigvalsh(Go))[::-1]
        kf = (w[:k].sum() - tucker1.kyfan_energy(Go, Sd)) / max(w[:k].sum(), 1e-300)
        T = torch.from_numpy(rng.random((3, m, n), dtype=np.float32) - 0.3)
        err = tsk.scw_error(T.cuda(), S, r).cpu().numpy()
        eo = oscw.scw_errors(T.numpy(), Sd, r)
        fro = np.linalg.norm(T.numpy().reshape(3, -1).astype(np.float64), axis=1)
        se = float(np.max(np.abs(err - eo) / (eo + 1e-6 * fro / 1e-4)))
        ok = ge <= 1e-5 and kf <= 1e-5 and np.all(np.abs(err - eo) <= 1e-4 * eo + 1e-6 * fro)
        bad += not ok
        print(f"{'ok ' if ok else 'BAD'} m={m} n={n} D={D} k={k} r={r} gramF={ge:.1e} kyfan={kf:.1e} scw={se:.1e} st={st}",
              flush=True)
    return bad


def suite_f_rows(ncase, rng):
    bad = 0
    for t in range(ncase):
        m = int(rng.integers(1, 100)) * 4; n = int(rng.integers(1, 100)) * 4; D = int(rng.integers(1, 10))
        A = torch.from_numpy(rng.random((D, m, n), dtype=np.float32) - 0.3)
        T = torch.from_numpy(rng.random((3, m, n), dtype=np.float32) - 0.3)
        msg = []
        ok = True
        # mode-2 Gram
        G2 = tsk.sketch_gram_mode2(A.cuda()).cpu().numpy()
        G2o = tucker2.mode2_gram(A.numpy())
        e = float(np.linalg.norm(G2 - G2o) / np.linalg.norm(G2o)); ok &= e <= 1e-5; msg.append(f"g2={e:.1e}")
        # two-sided: HOOI + SCW with the GPU's factors against the oracle's two-sided SCW
        k = int(rng.integers(1, min(m, 40) + 1)); l = int(rng.integers(1, min(n, 40) + 1))
        r = int(rng.integers(1, min(k, l) + 1))
        S, W, info, st = tsk.sketch_train_two_sided(A.cuda(), k, l, max_sweeps=3)
        e2 = tsk.two_sided_scw_error(T.cuda(), S, W, r).cpu().numpy()
        e2o = tucker2.two_sided_scw_errors(T.numpy(), S.cpu().double().numpy(), W.cpu().double().numpy(), r)
        fro = np.linalg.norm(T.numpy().reshape(3, -1).astype(np.float64), axis=1)
        ok2 = np.all(np.abs(e2 - e2o) <= 1e-4 * e2o + 1e-6 * fro); ok &= bool(ok2); msg.append(f"2scw={'ok' if ok2 else 'BAD'}")
        # matrix-free against its oracle (same start block)
        kk = int(rng.integers(1, min(m, 30) + 1)); ov = int(rng.integers(1, 20))
        p = min((kk + ov + 3) // 4 * 4, m)
        q = int(rng.integers(0, 3))
        if (q + 1) * p <= min(m, 256):
            om = datagen.start_block(m, p, t)
            Sm, lam, inf, stm = tsk.sketch_train_matrix_free(A.cuda(), kk, oversample=ov, power_iters=q, omega=om.cuda())
            So, th, K = omf.matrix_free_sketch(A.numpy(), kk, om.numpy(), q)
            e = float(np.max(np.abs(lam.cpu().numpy() - th[:kk])) / th[0]); ok &= e <= 1e-5; msg.append(f"mf={e:.1e}")
        # factors of sketch_apply_scw: A_hat = L R^T against the oracle's SCW
        k1 = int(rng.integers(1, min(m, 50) + 1)); r1 = int(rng.integers(1, min(k1, n, 64) + 1))
        S1, _, _, _ = tsk.sketch_train(A.cuda(), k1)
        L, R, sig = tsk.sketch_apply_scw(T.cuda(), S1, r1)
        Ah = torch.bmm(L, R.transpose(1, 2)).cpu().double().numpy()
        Aho = np.stack([oscw.scw(t, S1.cpu().double().numpy(), r1) for t in T.numpy()])
        e = float(np.max(np.linalg.norm((Ah - Aho).reshape(3, -1), axis=1) / fro)); ok &= e <= 1e-5; msg.append(f"fac={e:.1e}")
        bad += not ok
        print(("ok  " if ok else "BAD ") + f"m={m} n={n} D={D} k={k} l={l} r={r} kk={kk} p={p} q={q} k1={k1} r1={r1} " + " ".join(msg), flush=True)
    return bad


def suite_api(ncase, rng):
    bad = 0
    for t in range(ncase):
        m = int(rng.integers(2, 600)); n = int(rng.integers(1, 150)) * 4; D = int(rng.integers(2, 30))
        A = torch.from_numpy(rng.random((D, m, n), dtype=np.float32) - 0.3)
        msg, ok = [], True
        Gd, _ = tsk.sketch_gram(A.cuda())
        Gh, _ = tsk.sketch_gram(A)                     # host input (pageable), streamed by the library
        Gp, _ = tsk.sketch_gram(A.pin_memory())        # pinned
        eq = torch.equal(Gd.cpu(), Gh.cpu()) and torch.equal(Gd.cpu(), Gp.cpu()); ok &= eq; msg.append(f"host={'=' if eq else 'DIFF'}")
        h = int(rng.integers(1, D))
        Ga, _ = tsk.sketch_gram(A[:h].cuda())
        tsk.sketch_gram(A[h:].cuda(), G64=Ga, accumulate=True)
        e = float((Ga - Gd).norm() / Gd.norm()); ok &= e <= 1e-6; msg.append(f"acc={e:.1e}")
        G32 = torch.empty(m, m, dtype=torch.float32, device="cuda")
        G64b, _ = tsk.sketch_gram(A.cuda(), G32=G32)
        e = float((G32.double() - G64b).abs().max() / G64b.abs().max()); ok &= e <= 1e-6; msg.append(f"g32={e:.1e}")
        k = int(rng.integers(1, min(m, 40) + 1)); r = int(rng.integers(1, min(k, n, 64) + 1))
        S, lam, info, st = tsk.sketch_train(A.cuda(), k)
        T = torch.from_numpy(rng.random((4, m, n), dtype=np.float32) - 0.3)
        ed = tsk.scw_error(T.cuda(), S, r).cpu()
        eh = tsk.scw_error(T, S.cpu(), r)
        eq = torch.equal(ed, eh.cpu()); ok &= eq; msg.append(f"scw_host={'=' if eq else 'DIFF'}")
        L, R, sg = tsk.sketch_apply_scw(T.cuda(), S, r)
        ef = torch.linalg.norm((T.cuda().double() - torch.bmm(L.double(), R.double().transpose(1, 2))).reshape(4, -1), dim=1).cpu()
        # hybrid tolerance (reading c13): near an exactly-low-rank reconstruction both are at the 3xTF32 floor
        nrm = torch.linalg.norm(T.double().reshape(4, -1), dim=1)
        e = float(((ef - ed).abs() / (ed + 0.1 * nrm)).max())
        ok &= bool(((ef - ed).abs() <= 1e-5 * ed + 1e-6 * nrm).all()); msg.append(f"fac/err={e:.1e}")
        bad += not ok
        print(("ok  " if ok else "BAD ") + f"m={m} n={n} D={D} h={h} k={k} r={r} " + " ".join(msg), flush=True)
    return bad


def suite_mixed(ncase, rng):
    bad = 0
    for t in range(ncase):
        msg, ok = [], True
        # HOOI
        m = int(rng.integers(1, 80)) * 4; n = int(rng.integers(1, 80)) * 4; D = int(rng.integers(1, 8))
        k = int(rng.integers(1, min(m, 30) + 1)); l = int(rng.integers(1, min(n, 30) + 1))
        A = torch.from_numpy(rng.random((D, m, n), dtype=np.float32) - 0.3)
        S, W, info, st = tsk.sketch_train_two_sided(A.cuda(), k, l, max_sweeps=3, rel_tol=1e-14)
        Ad = A.numpy().astype(np.float64)
        So, Wo, hist_o, _ = tucker2.hooi_tucker2(Ad, k, l, max_iters=3, rel_tol=1e-14)
        rd = tucker2.tucker2_residual(Ad, S.cpu().double().numpy(), W.cpu().double().numpy())
        e = abs(rd - hist_o[-1]) / max(hist_o[-1], 1e-300); ok &= e <= 1e-5; msg.append(f"hooi={e:.1e}")
        # warm-started top-k from a perturbed exact sketch: same subspace energy
        m2 = int(rng.integers(257, 900)); n2 = int(rng.integers(1, 60)) * 4; D2 = int(rng.integers(2, 10))
        A2 = torch.from_numpy(rng.random((D2, m2, n2), dtype=np.float32) - 0.3)
        G, _ = tsk.sketch_gram(A2.cuda())
        k2 = int(rng.integers(1, 60))
        S0, lam0, _, _ = tsk.sketch_topk(G, k2)
        S_init = (S0 + 1e-2 * torch.randn_like(S0)).contiguous()
        S1, lam1, inf1, st1 = tsk.sketch_topk(G, k2, opts={"init_S": S_init})
        e = float((lam1 - lam0).abs().max() / lam0[0]); ok &= e <= 1e-6; msg.append(f"warm={e:.1e}")
        # split-K Gram: many thin slices
        m3 = int(rng.integers(2, 300)); n3 = int(rng.integers(1, 8)) * 4; D3 = int(rng.integers(100, 3000))
        A3 = torch.from_numpy(rng.random((D3, m3, n3), dtype=np.float32) - 0.3)
        G3, _ = tsk.sketch_gram(A3.cuda())
        A3d = A3.numpy().astype(np.float64)
        G3o = np.einsum("dik,djk->ij", A3d, A3d)
        e = float(np.linalg.norm(G3.cpu().numpy() - G3o) / np.linalg.norm(G3o)); ok &= e <= 1e-5; msg.append(f"splitK={e:.1e}")
        bad += not ok
        print(("ok  " if ok else "BAD ") + f"hooi m={m} n={n} D={D} k={k} l={l}; warm m={m2} k={k2}; gram m={m3} n={n3} D={D3} " +
              " ".join(msg), flush=True)
    return bad


def suite_spectra(ncase, rng):
    bad = 0
    kinds = ["flat", "geometric", "clustered", "rankdef", "dominant", "twogap", "steep"]
    for t in range(ncase):
        m = int(rng.integers(257, 1500)); k = int(rng.integers(1, 101))
        kind = kinds[t % len(kinds)]
        if kind == "flat":
            lam = 1.0 + 0.01 * rng.random(m)
        elif kind == "geometric":
            lam = 0.97 ** np.arange(m)
        elif kind == "clustered":
            lam = np.repeat(rng.random(m // 8 + 1) * 10, 8)[:m]
        elif kind == "rankdef":
            rk = int(rng.integers(1, 2 * k + 2)); lam = np.zeros(m); lam[:rk] = rng.random(rk) + 0.1
        elif kind == "dominant":
            lam = 1.0 + rng.random(m); lam[0] = 1e5
        elif kind == "steep":  # dominant mean, power-law top over a nearly flat bulk (C4-like, exaggerated)
            lam = 1.0 + 0.05 * rng.random(m); nt = int(rng.integers(2, 30))
            lam[1:nt + 1] += float(10 ** rng.uniform(2, 5)) * np.arange(1, nt + 1) ** -1.5; lam[0] = 1e6
        else:
            lam = np.concatenate([np.full(k, 10.0), np.full(m - k, 1.0)]) + 1e-3 * rng.random(m)
        U, _ = torch.linalg.qr(torch.randn(m, m, dtype=torch.float64, device="cuda"))
        L = torch.tensor(lam, dtype=torch.float64, device="cuda")
        G = (U * L) @ U.T
        G = 0.5 * (G + G.T)
        t0 = time.time()
        with np.errstate(all="ignore"):
            import warnings
            with warnings.catch_warnings(record=True) as wl:
                warnings.simplefilter("always")
                S, lmb, info, st = tsk.sketch_topk(G.contiguous(), k, opts=None)
        torch.cuda.synchronize()
        ms = (time.time() - t0) * 1e3
        ws = np.sort(lam)[::-1]
        Sd = S.double()
        kf = float(torch.einsum("ci,ij,cj->", Sd, G, Sd))
        dfc = (ws[:k].sum() - kf) / ws[:k].sum()
        orth = float(torch.linalg.norm(Sd @ Sd.T - torch.eye(k, dtype=torch.float64, device="cuda")))
        ok = dfc <= 1e-6 and orth <= 1e-5
        bad += not ok
        print(("ok  " if ok else "BAD ") + f"{kind:9s} m={m} k={k} st={st} warn={len(wl)} products={info.iters} "
              f"deficit={dfc:.1e} orth={orth:.1e} {ms:.0f} ms", flush=True)
    return bad


def suite_limits(ncase, rng):
    bad = 0
    for t in range(ncase):
        m = int(rng.integers(33, 80)) * 4; n = int(rng.integers(33, 80)) * 4
        k = int(rng.integers(90, min(m, 128) + 1)); r = int(rng.integers(1, min(k, 64) + 1))
        T = torch.from_numpy(rng.random((4, m, n), dtype=np.float32) - 0.3)
        S = orth_rows(rng, k, m)
        e = tsk.scw_error(T.cuda(), S.cuda(), r).cpu().numpy()
        eo = oscw.scw_errors(T.numpy(), S.double().numpy(), r)
        fro = np.linalg.norm(T.numpy().reshape(4, -1).astype(np.float64), axis=1)
        ok1 = bool(np.all(np.abs(e - eo) <= 1e-4 * eo + 1e-6 * fro))
        k2 = int(rng.integers(60, min(m, 116) + 1)); l2 = int(rng.integers(60, min(n, 116) + 1)); r2 = int(rng.integers(1, min(k2, l2, 64) + 1))
        S2 = orth_rows(rng, k2, m); W2 = orth_rows(rng, l2, n)
        e2 = tsk.two_sided_scw_error(T.cuda(), S2.cuda(), W2.cuda(), r2).cpu().numpy()
        e2o = tucker2.two_sided_scw_errors(T.numpy(), S2.double().numpy(), W2.double().numpy(), r2)
        ok2 = bool(np.all(np.abs(e2 - e2o) <= 1e-4 * e2o + 1e-6 * fro))
        ok = ok1 and ok2
        bad += not ok
        print(("ok  " if ok else "BAD ") + f"m={m} n={n} k={k} r={r} scw={float(np.max(np.abs(e - eo) / eo)):.1e}; "
              f"k2={k2} l2={l2} r2={r2} two-sided={float(np.max(np.abs(e2 - e2o) / e2o)):.1e}", flush=True)
    return bad


SUITES = {"core": suite_core, "f_rows": suite_f_rows, "api": suite_api, "mixed": suite_mixed,
          "spectra": suite_spectra, "limits": suite_limits}

if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    names = list(SUITES) if not args or args[0] == "all" else [args[0]]
    ncase = int(args[1]) if len(args) > 1 else 10
    seed = int(args[2]) if len(args) > 2 else 0
    total = 0
    for nm in names:
        print(f"== {nm}", flush=True)
        total += SUITES[nm](ncase, np.random.default_rng(seed))
    print("failures:", total)
