"""Rank-deficient Grams (rank D*n < k): the eigensolver must still return an orthonormal S with the optimal Ky Fan energy (developer check)."""
import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch, paper_2209_14637_b200 as tsk
from oracle import tucker1
for (m, n, D, k) in [(500, 8, 1, 20), (300, 4, 2, 12), (1000, 12, 1, 40), (64, 4, 1, 10), (257, 4, 3, 30)]:
    g = torch.Generator().manual_seed(m)
    A = torch.rand(D, m, n, generator=g) - 0.3
    G, _ = tsk.sketch_gram(A.cuda())
    try:
        S, lam, info, st = tsk.sketch_topk(G, k)
        Sd = S.cpu().double().numpy(); Go = tucker1.mode1_gram(A.numpy())
        w = np.sort(np.linalg.eigvalsh(Go))[::-1]
        print(m, n, D, k, "st", st, "orth", np.linalg.norm(Sd @ Sd.T - np.eye(k)), "kyfan def", (w[:k].sum() - tucker1.kyfan_energy(Go, Sd)) / w[:k].sum(), "iters", info.iters)
    except Exception as e:
        print(m, n, D, k, "ERROR", e)
