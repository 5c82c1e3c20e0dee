"""Jacobi eigensolver probe: accuracy vs numpy, sweeps, time (developer script)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402

def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

for p, B, kind in [(20, 1, "rand"), (60, 1, "rand"), (90, 1, "rand"), (90, 1, "neardiag"), (128, 1, "rand"), (150, 1, "rand"), (60, 500, "rand")]:
    rng = np.random.default_rng(p)
    Hs = []
    for _ in range(B):
        X = rng.standard_normal((p, p))
        if kind == "rand":
            ev = np.exp(rng.uniform(-8, 8, p))
            Q = np.linalg.qr(X)[0]
        else:
            ev = np.exp(rng.uniform(-8, 8, p)); Q = np.linalg.qr(np.eye(p) + 1e-3 * X)[0]
        Hs.append((Q * ev) @ Q.T)
    H = torch.tensor(np.array(Hs), device="cuda")
    W, lam, sw = tsk.tsk_eig_probe(H)
    ms = timeit(lambda: tsk.tsk_eig_probe(H))
    Hn = H[0].cpu().numpy(); Wn = W[0].cpu().numpy(); ln = lam[0].cpu().numpy()
    ref = np.sort(np.linalg.eigvalsh(Hn))[::-1]
    res = np.linalg.norm(Hn @ Wn - Wn * ln) / np.linalg.norm(Hn)
    orth = np.linalg.norm(Wn.T @ Wn - np.eye(p))
    print(f"p={p} B={B} {kind}: {ms*1e3:.0f} us  sweeps={sw[:4].tolist()}  lam relerr={np.max(np.abs(ln-ref))/ref[0]:.2e} resid={res:.2e} orth={orth:.2e}", flush=True)
