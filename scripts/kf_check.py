"""Ky Fan deficit and Ritz-value accuracy of the GPU sketch at full C4 against fp64 eigh of the GPU Gram (developer check)."""
import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch, datagen, paper_2209_14637_b200 as tsk
from oracle import tucker1
c = datagen.CONFIGS["C4"]
A = datagen.generate(c, "train", device="cuda")
G = torch.empty(c.m, c.m, dtype=torch.float64, device="cuda")
opts = {"tol_active": 1} if "--active" in sys.argv else None
S, lam, info, st = tsk.sketch_train(A, c.k, opts=opts, G64_out=G)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); S, lam, info, st = tsk.sketch_topk(G, c.k, opts=opts); e1.record(); torch.cuda.synchronize()
print("topk ms", e0.elapsed_time(e1), "products", info.iters, "status", st)
Gg = G.cpu().numpy(); w = np.sort(np.linalg.eigvalsh(Gg))[::-1]
Sd = S.cpu().double().numpy()
kf = tucker1.kyfan_energy(Gg, Sd)
print("kyfan deficit rel", (w[:c.k].sum() - kf) / w[:c.k].sum(), "lam err/top", np.max(np.abs(lam.cpu().numpy() - w[:c.k])) / w[0], "max_resid", info.max_resid)
print("deficit excl top", (w[1:c.k].sum() - (kf - w[0])) / w[1:c.k].sum())
