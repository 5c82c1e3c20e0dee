import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402
p = int(sys.argv[1]) if len(sys.argv) > 1 else 90
rng = np.random.default_rng(0)
Q = np.linalg.qr(rng.standard_normal((p, p)))[0]
H = torch.tensor(((Q * np.exp(rng.uniform(-8, 8, p))) @ Q.T)[None], device="cuda")
for _ in range(2):
    W, lam, sw = tsk.tsk_eig_probe(H)
torch.cuda.synchronize(); print("sweeps", sw.tolist())
