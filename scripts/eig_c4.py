"""Eigensolver behaviour at C4 (m = 1080, k = 60): python scripts/eig_c4.py (TSK_EIG_TRACE=1 for the
per-iteration lines).  Times 5 calls of sketch_topk on the C4 Gram."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402
c = datagen.CONFIGS["C4"]
A = datagen.generate(c, "train", device="cuda")
G, _ = tsk.sketch_gram(A)
del A
for i in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    S, lam, info, st = tsk.sketch_topk(G, c.k)
    e1.record()
    torch.cuda.synchronize()
    print(f"topk: {e0.elapsed_time(e1):.2f} ms products={info.iters} max_resid={info.max_resid:.2e} status={st}", flush=True)
