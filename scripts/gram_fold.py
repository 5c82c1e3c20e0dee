"""Pair-Gram fold interval (TSK_PAIR_FOLD, chains between fp64 folds of the fp32 register sums):
time and Gram relative Frobenius error against an fp64 torch reference, on the C3/C4 frame-like
streams (D frames).  python scripts/gram_fold.py C4 [D]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
c = datagen.CONFIGS[name]
D = int(sys.argv[2]) if len(sys.argv) > 2 else c.D_train
A = datagen.generate(c, "train", 0, D, device="cuda")
Gr = torch.zeros(c.m, c.m, dtype=torch.float64, device="cuda")
for d0 in range(0, D, 50):
    Ad = A[d0:d0 + 50].double()
    Gr += torch.einsum("dik,djk->ij", Ad, Ad)
del Ad
G = torch.empty(c.m, c.m, dtype=torch.float64, device="cuda")
tsk.sketch_gram(A, G64=G)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    tsk.sketch_gram(A, G64=G)
e1.record()
torch.cuda.synchronize()
err = (torch.linalg.norm(G - Gr) / torch.linalg.norm(Gr)).item()
print(f"{name} D={D} fold={os.environ.get('TSK_PAIR_FOLD', 'default')}: {e0.elapsed_time(e1) / 3:.2f} ms  "
      f"Gram rel-F error {err:.2e}", flush=True)
