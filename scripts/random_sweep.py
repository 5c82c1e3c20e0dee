"""Randomised robustness sweep (developer check): random shapes for the Gram, the sketch and SCW against
the float64 oracle.  python scripts/random_sweep.py [n_cases] [seed]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402
from oracle import scw as oscw, tucker1  # noqa: E402

ncase = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
big = "--big" in sys.argv  # m up to 1500 (subspace-iteration eigensolver), k up to 100
bad = 0
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
print("failures:", bad)
