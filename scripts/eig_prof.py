"""Profile helper: one sketch_topk at C4 and syev probes at p = 76 / 128 between cudaProfilerStart/Stop
(ncu --profile-from-start off).  python scripts/eig_prof.py"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402
name = os.environ.get("CFG", "C4")
c = datagen.CONFIGS[name]
G = torch.zeros(c.m, c.m, dtype=torch.float64, device="cuda")
buf = torch.empty(200, c.m, c.n, dtype=torch.float32, device="cuda")
for d0 in range(0, c.D_train, 200):
    d1 = min(c.D_train, d0 + 200)
    datagen.generate(c, "train", d0, d1, device="cuda", out=buf[: d1 - d0])
    tsk.sketch_gram(buf[: d1 - d0], G64=G, accumulate=d0 > 0)
del buf
rng = np.random.default_rng(0)
Hs = []
for p in (76, 128):
    Q = np.linalg.qr(rng.standard_normal((p, p)))[0]
    Hs.append(torch.tensor((Q * np.exp(rng.uniform(-8, 8, p))) @ Q.T, device="cuda"))
tsk.sketch_topk(G, c.k)
for H in Hs:
    tsk.tsk_syev_probe(H)
torch.cuda.synchronize()
torch.cuda.profiler.start()
tsk.sketch_topk(G, c.k)
for H in Hs:
    tsk.tsk_syev_probe(H)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
