"""Microbenchmarks / hardware behaviour probes for the Gram kernel (developer script)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def tf32_trunc(x):
    b = x.view(np.uint32) & np.uint32(0xFFFFE000)
    return b.view(np.float32)


def tf32_rn(x):
    b = x.view(np.uint32).astype(np.uint64)
    b = (b + 0x1000) & 0xFFFFE000  # round half away (magnitude), ignoring overflow corner cases
    return b.astype(np.uint32).view(np.float32)


def main():
    # ---- operand conversion: does kind::tf32 truncate or round fp32 inputs?
    torch.manual_seed(0)
    A = torch.rand(4, 128, 64) + 0.5
    Gg = tsk.tsk_gram_probe(A.cuda(), mode=3, chain=1).cpu().numpy()
    a = A.numpy()
    for name, f in (("trunc", tf32_trunc), ("rn", tf32_rn), ("exact", lambda x: x)):
        h = f(a.copy()).astype(np.float64)
        G = sum(x @ x.T for x in h)
        print(f"operand model {name:5s}: relF(gpu - model) = {np.linalg.norm(Gg - G) / np.linalg.norm(G):.3e}")
    # ---- throughput breakdown at C4 shape (random data)
    m, n, D = 1080, 1920, 2000
    X = torch.rand(D, m, n, device="cuda")
    alg = m * (m + 1) * n * D
    Xs = X[:200].contiguous()
    Xd = Xs.double()
    Gref = torch.einsum("dij,dkj->ik", Xd, Xd)
    for ch in (1, 2, 4, 8, 16):
        Gs = tsk.tsk_gram_probe(Xs, mode=0, chain=ch)
        print(f"accuracy chain={ch}: relF={float((Gs - Gref).norm() / Gref.norm()):.3e}", flush=True)
    del Xd
    for mode, label in ((0, "split 3xTF32"), (1, "raw tiles, 3 products (no transform)"),
                        (3, "raw tiles, 1 product")):
        for ch in (1, 2, 4, 8):
            ms = timeit(lambda: tsk.tsk_gram_probe(X, mode=mode, chain=ch))
            print(f"mode={mode} ({label}) chain={ch}: {ms:.2f} ms  alg {alg / ms / 1e9:.0f} TF/s  "
                  f"issued {(3 if mode in (0, 1) else 1) * alg / ms / 1e9:.0f} TF/s", flush=True)


if __name__ == "__main__":
    main()
