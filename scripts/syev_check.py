"""Developer check of the Rayleigh-Ritz eigensolver (syev.cu) against numpy: accuracy and time."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402


def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


rng = np.random.default_rng(0)
for p, kind in [(20, "rand"), (60, "rand"), (76, "rand"), (76, "c4like"), (116, "c5like"), (128, "rand"),
                (160, "rand"), (200, "rand"), (256, "rand"), (76, "cluster"), (76, "null")]:
    if kind == "rand":
        ev = np.exp(rng.uniform(-8, 8, p))
    elif kind == "c4like":
        ev = np.r_[1.3e6 * 0.9 ** np.arange(10), 6e4 + 50 * rng.standard_normal(p - 10)]
    elif kind == "c5like":
        ev = 865 + 0.5 * rng.standard_normal(p)
    elif kind == "cluster":
        ev = np.r_[np.ones(5) * 3.0, rng.uniform(0, 2, p - 5)]
    else:
        ev = np.r_[rng.uniform(1, 2, p // 2), np.zeros(p - p // 2)]
    Q = np.linalg.qr(rng.standard_normal((p, p)))[0]
    H = (Q * ev) @ Q.T
    H = 0.5 * (H + H.T)
    Hd = torch.tensor(H, device="cuda")
    W, lam, flag = tsk.tsk_syev_probe(Hd)
    ms = timeit(lambda: tsk.tsk_syev_probe(Hd))
    Wn, ln = W.cpu().numpy(), lam.cpu().numpy()
    ref = np.sort(np.linalg.eigvalsh(H))[::-1]
    res = np.linalg.norm(H @ Wn - Wn * ln) / np.linalg.norm(H)
    orth = np.max(np.abs(Wn.T @ Wn - np.eye(p)))
    print(f"p={p:3d} {kind:8s}: {ms * 1e3:7.1f} us  lam relerr={np.max(np.abs(ln - ref)) / abs(ref[0]):.1e} "
          f"resid={res:.1e} orth={orth:.1e} flag={int(flag.item())}", flush=True)
