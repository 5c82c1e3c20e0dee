"""Randomised sweep at the size limits (developer check): SCW with k in [90, 128] (the chol-basis /
Jacobi-fallback boundary at 116), r up to 64, two-sided SCW with k, l up to 116; against the oracle.
python scripts/random_sweep6.py [n_cases] [seed]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402
from oracle import scw as oscw, tucker2  # noqa: E402

def orth_rows(rng, k, m):
    q, _ = np.linalg.qr(rng.standard_normal((m, k)))
    return torch.tensor(q.T.copy(), dtype=torch.float32)

ncase = int(sys.argv[1]) if len(sys.argv) > 1 else 10
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
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
print("failures:", bad)
