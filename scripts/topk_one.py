"""Gram + top-k at a config, for launch-list profiling: python scripts/topk_one.py C4 [D]"""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402
c = datagen.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
D = int(sys.argv[2]) if len(sys.argv) > 2 else 200
A = datagen.generate(c, "train", 0, D, device="cuda")
G, _ = tsk.sketch_gram(A)
torch.cuda.synchronize()
t = time.time()
S, lam, info, st = tsk.sketch_topk(G, c.k)
torch.cuda.synchronize()
print(f"topk {1e3*(time.time()-t):.1f} ms info={info.as_dict()}")
