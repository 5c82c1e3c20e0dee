"""Pythagorean SCW error (reading c17) vs the dense residual: run once per mode (env TSK_SCW_DENSE=1 /
TSK_SCW_PYTH_TAU=0), saving the per-matrix errors and ||A||_F^2 of the C1-C4 test streams to
gpurun_out/pyth_<mode>_<cfg>.npz.  python scripts/scw_pyth_check.py <mode> [C1 C2 C3 C4]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402

mode = sys.argv[1]
for name in sys.argv[2:] or ["C1", "C2", "C3", "C4"]:
    c = datagen.CONFIGS[name]
    T = datagen.generate(c, "test", device="cuda")
    q, _ = np.linalg.qr(np.random.default_rng(0).standard_normal((c.m, c.k)))
    S = torch.tensor(q.T.copy(), dtype=torch.float32, device="cuda")
    e = tsk.scw_error(T, S, c.r).cpu().numpy()
    nrm2 = (T.double() ** 2).sum(dim=(1, 2)).cpu().numpy()
    os.makedirs("gpurun_out", exist_ok=True)
    np.savez(f"gpurun_out/pyth_{mode}_{name}.npz", e=e, nrm2=nrm2)
    print(mode, name, "err^2/|A|^2 min %.3e max %.3e" % ((e ** 2 / nrm2).min(), (e ** 2 / nrm2).max()), flush=True)
