"""Profile helper: syev probe at p (argv[1]) repeated (ncu sampling) -- python scripts/syev_rep.py 76 20"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402
p = int(sys.argv[1]); reps = int(sys.argv[2])
rng = np.random.default_rng(0)
Q = np.linalg.qr(rng.standard_normal((p, p)))[0]
H = torch.tensor((Q * np.exp(rng.uniform(-8, 8, p))) @ Q.T, device="cuda")
for _ in range(reps):
    tsk.tsk_syev_probe(H)
torch.cuda.synchronize()
