"""scw_error at C4 with the trained sketch (as in bench.py) against a random orthonormal S: time, and how
many matrices take the dense-residual fallback (errors equal under TSK_SCW_DENSE, reading c17).
python scripts/scw_trained.py [C4]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
c = datagen.CONFIGS[name]
G = torch.zeros(c.m, c.m, dtype=torch.float64, device="cuda")
buf = torch.empty(200, c.m, c.n, device="cuda")
for d0 in range(0, c.D_train, 200):
    d1 = min(c.D_train, d0 + 200)
    datagen.generate(c, "train", d0, d1, device="cuda", out=buf[: d1 - d0])
    tsk.sketch_gram(buf[: d1 - d0], G64=G, accumulate=d0 > 0)
del buf
S, lam, info, st = tsk.sketch_topk(G, c.k)
T = datagen.generate(c, "test", device="cuda")
q, _ = np.linalg.qr(np.random.default_rng(0).standard_normal((c.m, c.k)))
Sr = torch.tensor(q.T.copy(), dtype=torch.float32, device="cuda")
for lab, SS in (("trained", S), ("random", Sr)):
    err = torch.empty(c.D_test, dtype=torch.float64, device="cuda")
    for _ in range(2):
        tsk.scw_error(T, SS, c.r, out=err)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); tsk.scw_error(T, SS, c.r, out=err); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    nrm2 = (T.double() ** 2).sum(dim=(1, 2))
    frac = (err ** 2 / nrm2)
    print(f"{lab}: scw_error {min(ts):.3f} ms; err^2/||A||^2 min {frac.min().item():.2e} median "
          f"{frac.median().item():.2e}; below tau 3e-3: {(frac < 3e-3).sum().item()} of {c.D_test}", flush=True)
