import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_2209_14637_b200 as tsk  # noqa
c = datagen.CONFIGS["C4"]
A = datagen.generate(c, "train", 0, 100, device="cuda")
G, _ = tsk.sketch_gram(A)
S, lam, info, st = tsk.sketch_topk(G, c.k, opts={"max_iters": 6})
torch.cuda.synchronize(); print("ok", info.iters)
