"""Eigensolver robustness across spectra (developer check): G = U diag(lambda) U^T with flat, geometric,
clustered, rank-deficient and dominant-plus-flat spectra, m in [257, 1500]: Ky Fan deficit, orthonormality
and status of sketch_topk.  python scripts/random_sweep5.py [n_cases] [seed]"""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402

ncase = int(sys.argv[1]) if len(sys.argv) > 1 else 12
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
kinds = ["flat", "geometric", "clustered", "rankdef", "dominant", "twogap"]
if "--dominant" in sys.argv:
    kinds = ["dominant"]
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
            S, lmb, info, st = tsk.sketch_topk(G.contiguous(), k, opts={"tol_active": 1} if "--active" in sys.argv else None)
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
print("failures:", bad)
