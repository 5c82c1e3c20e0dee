"""Developer check: sketch_topk on the seed-4 random shape of tests/test_gpu_random_shapes.py (TSK_EIG_TRACE=1)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402
from oracle import tucker1  # noqa: E402
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rng = np.random.default_rng(1000 + seed)
m = int(rng.integers(2, 700)); n = int(rng.integers(1, 200)) * 4; D = int(rng.integers(1, 12))
A = torch.from_numpy(rng.random((D, m, n), dtype=np.float32) - 0.3)
G, _ = tsk.sketch_gram(A.cuda())
k = int(rng.integers(1, min(m, 60) + 1))
print("m", m, "n", n, "D", D, "k", k, flush=True)
S, lam, info, st = tsk.sketch_topk(G, k)
Go = tucker1.mode1_gram(A.numpy())
w = np.sort(np.linalg.eigvalsh(Go))[::-1]
print("deficit", (w[:k].sum() - tucker1.kyfan_energy(Go, S.cpu().double().numpy())) / w[:k].sum(), "status", st, "iters", info.iters)
print("lam", lam.cpu().numpy()[:5], "true", w[:5], "rank-ish", int((w > 1e-10 * w[0]).sum()))
