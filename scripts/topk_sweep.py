"""Eigensolver iterations/time vs oversampling at a config (developer script)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402
c = datagen.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
D = int(sys.argv[2]) if len(sys.argv) > 2 else 200
A = datagen.generate(c, "train", 0, D, device="cuda")
G, _ = tsk.sketch_gram(A)
import numpy as np
from oracle import tucker1
Gn = G.cpu().numpy()
lam_g = np.sort(np.linalg.eigvalsh(Gn))[::-1]
tols = [float(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [1e-6]
for ov in [int(x) for x in sys.argv[3].split(",")]:
  for tol in tols:
    for rep in range(2):
        torch.cuda.synchronize(); t = time.time()
        S, lam, info, st = tsk.sketch_topk(G, c.k, opts={"oversample": ov, "tol": tol})
        torch.cuda.synchronize()
    Sg = S.cpu().double().numpy()
    dfc = (lam_g[:c.k].sum() - tucker1.kyfan_energy(Gn, Sg)) / lam_g[:c.k].sum()
    print(f"oversample={ov} tol={tol:.0e}: {1e3*(time.time()-t):.1f} ms iters={info.iters} res={info.max_resid:.2e} "
          f"st={st} kyfan_deficit={dfc:.2e}", flush=True)
