"""A/B timing of Gram kernel variants at C4 shape (developer script): python scripts/gram_ab.py"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402

def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

m, n, D = 1080, 1920, 2000
X = torch.rand(D, m, n, device="cuda")
alg = m * (m + 1) * n * D
Xs = X[:200].contiguous(); Xd = Xs.double(); Gref = torch.einsum("dij,dkj->ik", Xd, Xd); del Xd
for mode in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,4").split(",")]:
    for ch in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]:
        ms = timeit(lambda: tsk.tsk_gram_probe(X, mode=mode, chain=ch))
        e = float((tsk.tsk_gram_probe(Xs, mode=mode, chain=ch) - Gref).norm() / Gref.norm())
        print(f"mode={mode} chain={ch}: {ms:.2f} ms  alg {alg/ms/1e9:.0f} TF/s  relF(200)={e:.2e}", flush=True)
