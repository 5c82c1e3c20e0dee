"""Profile helper: one scw_error call on the 500 C4 test matrices between cudaProfilerStart/Stop, plus
its CUDA-event time.  python scripts/scw_prof.py [C4]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
c = datagen.CONFIGS[name]
T = datagen.generate(c, "test", device="cuda")
q, _ = np.linalg.qr(np.random.default_rng(0).standard_normal((c.m, c.k)))
S = torch.tensor(q.T.copy(), dtype=torch.float32, device="cuda")
err = torch.empty(c.D_test, dtype=torch.float64, device="cuda")
for _ in range(2):
    tsk.scw_error(T, S, c.r, out=err)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); tsk.scw_error(T, S, c.r, out=err); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"scw_error {name} B={c.D_test}: {min(ts):.3f} ms (min of 5), {np.median(ts):.3f} median", flush=True)
torch.cuda.profiler.start()
tsk.scw_error(T, S, c.r, out=err)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
