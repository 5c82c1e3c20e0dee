"""Per-chunk timeline of cluster 0 of the pair Gram (TSK_PAIR_TRACE): python scripts/gram_pair_trace.py mode D"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
D = int(sys.argv[2]) if len(sys.argv) > 2 else 200
X = torch.rand(D, 1080, 1920, device="cuda")
tsk.tsk_gram_probe(X, mode=mode)
os.environ["TSK_PAIR_TRACE"] = "/tmp/trace.bin"
tsk.tsk_gram_probe(X, mode=mode)
torch.cuda.synchronize()
raw = np.fromfile("/tmp/trace.bin", dtype=np.uint64).astype(np.int64)
per = raw[-296:].reshape(148, 2)
t = raw[:-296].reshape(11, -1)
per = per[per[:, 0] > 0]
t0 = per[:, 0].min()
print("cluster start (us):", np.round((per[:, 0] - t0) / 1e3, 1).tolist())
print("cluster end   (us):", np.round((per[:, 1] - t0) / 1e3, 1).tolist())
n = int((t[2] > 0).sum())
t = t[:, 20:min(n, 400)]
base = t[1]
names = ["mma_start", "mma_lfull_ok", "mma_committed", "tf0_rfull_ok", "tf0_lempty_ok", "tf0_arrive",
         "tf1_rfull_ok", "tf1_lempty_ok", "tf1_arrive", "epi_accf_ok", "epi_arrive"]
print(f"mode {mode}: chunks traced {n}; per-chunk MMA period {np.median(np.diff(t[1]))/8:.0f} ns")
full = np.fromfile("/tmp/trace.bin", dtype=np.uint64).astype(np.int64)[:-296].reshape(11, -1)[1]
full = full[full > 0]
seg = np.diff(full) / 8
print("span of samples (us):", (full[-1]-full[0])/1e3, " n samples", len(full), " largest gaps (us):", np.round(np.sort(np.diff(full))[-12:]/1e3,1).tolist(), " gap positions:", np.argsort(np.diff(full))[-12:].tolist())
print("period (ns/chunk) in consecutive blocks of 256 samples:", [int(np.median(seg[i:i+256])) for i in range(0, len(seg), 256)])
ep = np.fromfile("/tmp/trace.bin", dtype=np.uint64).astype(np.int64)[:-296].reshape(11, -1)
ok = (ep[9] > 0) & (ep[10] > 0)
print("epilogue per chain: drain duration median ns", np.median((ep[10]-ep[9])[ok]), " accf period median ns", np.median(np.diff(ep[9][ok])))
for i, nm in enumerate(names[:9]):
    print(f"{nm:15s} rel. to mma_lfull_ok of same chunk: median {np.median(t[i] - base):8.0f} ns  p10 {np.percentile(t[i]-base,10):8.0f}  p90 {np.percentile(t[i]-base,90):8.0f}")
