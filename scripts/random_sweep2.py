"""Randomised robustness sweep of the f-row entry points (developer check): mode-2 Gram, HOOI +
two-sided SCW, the matrix-free sketch, sketch_apply_scw factors -- against the float64 oracle.
python scripts/random_sweep2.py [n_cases] [seed]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402
from oracle import matrix_free as omf, scw as oscw, tucker1, tucker2  # noqa: E402

ncase = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
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
print("failures:", bad)
