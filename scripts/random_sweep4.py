"""Randomised sweep (developer check): HOOI against the oracle HOOI on random shapes, warm-started top-k,
and split-K Grams with many slices.  python scripts/random_sweep4.py [n_cases] [seed]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402
from oracle import tucker1, tucker2  # noqa: E402

ncase = int(sys.argv[1]) if len(sys.argv) > 1 else 12
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
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
print("failures:", bad)
