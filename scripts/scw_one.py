"""One SCW-error call at C4 shape (500 test matrices) for profiling: python scripts/scw_one.py [B]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402
B = int(sys.argv[1]) if len(sys.argv) > 1 else 500
m, n, k, r = 1080, 1920, 60, 30
g = torch.Generator(device="cuda").manual_seed(0)
T = torch.rand(B, m, n, device="cuda", generator=g)
S = torch.linalg.qr(torch.randn(m, k, device="cuda", generator=g, dtype=torch.float64))[0].T.contiguous().float()
for _ in range(2):
    e = tsk.scw_error(T, S, r)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
e = tsk.scw_error(T, S, r)
ev1.record()
torch.cuda.synchronize()
print(f"scw_error B={B}: {ev0.elapsed_time(ev1):.2f} ms")
