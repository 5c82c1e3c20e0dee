"""One syev probe at p (argv[1], default 76) -- for compute-sanitizer runs."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402
p = int(sys.argv[1]) if len(sys.argv) > 1 else 76
rng = np.random.default_rng(0)
Q = np.linalg.qr(rng.standard_normal((p, p)))[0]
H = torch.tensor((Q * np.exp(rng.uniform(-8, 8, p))) @ Q.T, device="cuda")
W, lam, flag = tsk.tsk_syev_probe(H)
torch.cuda.synchronize()
print("ok", p, float(lam[0]), int(flag))
