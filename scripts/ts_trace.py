"""Per-chunk timeline of CTA 0 of the TS tensor-core kernel (TSK_TS_TRACE) during one C4 scw_error: for each
launch, the chunk period and where a chunk waits (TMA issue -> transform rfull_ok -> lempty_ok -> arrive ->
MMA lfull_ok -> MMA issued).  python scripts/ts_trace.py [C4]"""
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
tsk.scw_error(T, S, c.r, out=err)
torch.cuda.synchronize()
path = "/tmp/ts_trace.bin"
if os.path.exists(path):
    os.remove(path)
os.environ["TSK_TS_TRACE"] = path
tsk.scw_error(T, S, c.r, out=err)
torch.cuda.synchronize()
raw = np.fromfile(path, dtype=np.uint64).astype(np.int64).reshape(-1, 8, 8192)
names = ["tma_issue", "mma_lfull_ok", "mma_issued", "tf_rfull_ok", "tf_lempty_ok", "tf_arrive"]
for li, t in enumerate(raw):
    n = int((t[2] > 0).sum())
    if n < 50:
        continue
    t = t[:, 10:n - 5]
    per = np.median(np.diff(t[2]))
    print(f"launch {li}: chunks {n}, MMA issue period median {per:.0f} ns, p10 {np.percentile(np.diff(t[2]), 10):.0f} "
          f"p90 {np.percentile(np.diff(t[2]), 90):.0f}")
    base = t[1]
    for i, nm in enumerate(names):
        d = t[i] - base
        print(f"   {nm:14s} rel. to mma_lfull_ok of the same chunk: median {np.median(d):9.0f} ns  "
              f"p10 {np.percentile(d, 10):9.0f}  p90 {np.percentile(d, 90):9.0f}")
    print(f"   transform busy (arrive - lempty_ok) median {np.median(t[5] - t[4]):.0f} ns; "
          f"rfull wait (rfull_ok - prev arrive) median {np.median(t[3][1:] - t[5][:-1]):.0f} ns; "
          f"lempty wait median {np.median(t[4] - t[3]):.0f} ns; TMA issue -> rfull_ok median "
          f"{np.median(t[3] - t[0]):.0f} ns")
