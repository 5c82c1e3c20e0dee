"""Batched Jacobi timing (developer script): python scripts/jacobi_time.py"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402
g = torch.Generator(device="cuda").manual_seed(0)
for (p, B) in [(int(a.split("x")[0]), int(a.split("x")[1])) for a in (sys.argv[1:] or ["76x1", "60x1", "60x500", "20x100", "40x200"])]:
    X = torch.randn(B, p, 3 * p, device="cuda", dtype=torch.float64, generator=g)
    H = X @ X.transpose(1, 2)
    tsk.tsk_eig_probe(H)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        W, lam, sw = tsk.tsk_eig_probe(H)
    e1.record()
    torch.cuda.synchronize()
    print(f"p={p} B={B}: {e0.elapsed_time(e1) / 5:.3f} ms  sweeps max {int(sw.max())}", flush=True)
