"""Eigensolver behaviour at C5 (m = 4096, k = 100): python scripts/eig_c5.py [D] (TSK_EIG_TRACE=1 for
per-iteration lines).  Builds G from D C5 training matrices, runs sketch_topk, reports products,
residual and time, and the Ky Fan deficit against a torch fp64 eigh of the same G (a dev check)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402
D = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
c = datagen.CONFIGS["C5"]
G = torch.zeros(c.m, c.m, dtype=torch.float64, device="cuda")
for d0 in range(0, D, 250):
    A = datagen.generate(c, "train", d0, min(D, d0 + 250), device="cuda")
    tsk.sketch_gram(A, G64=G, accumulate=d0 > 0)
    del A
torch.cuda.synchronize()
ov = int(os.environ.get("OVERSAMPLE", "0"))
opts = {"oversample": ov} if ov else None
tsk.sketch_topk(G, c.k, opts=opts)
torch.cuda.synchronize()
t = time.time()
S, lam, info, st = tsk.sketch_topk(G, c.k, opts=opts)
torch.cuda.synchronize()
el = time.time() - t
w = torch.linalg.eigvalsh(G)
top = w.flip(0)[: c.k].sum()
Sd = S.double()
ky = torch.einsum("ci,ij,cj->", Sd, G, Sd)
print(f"D={D} status={st} products={info.iters} max_resid={info.max_resid:.3e} time={el*1e3:.1f} ms "
      f"kyfan_deficit={float((top - ky) / top):.3e} gap={float(w.flip(0)[c.k-1] / w.flip(0)[c.k]):.5f} "
      f"lam1={float(w[-1]):.4e} lam_k={float(w.flip(0)[c.k-1]):.4e} froG/lam1={float(G.norm() / w[-1]):.2f}")
