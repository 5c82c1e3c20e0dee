"""Developer timing sweep of the CTA-pair Gram at C4 shape: python scripts/gram_pair_time.py"""
import os
import sys

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


m, n, D = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1080,1920,2000").split(","))
X = torch.rand(D, m, n, device="cuda")
alg = m * (m + 1) * n * D
runs = [(16, 4, 0, None), (0, 4, 0, None), (32, 4, 0, None), (36, 4, 0, None), (32, 8, 0, None),
        (32, 4, 0, "37")]
if len(sys.argv) > 2:
    runs = [tuple(int(v) if i < 3 else (v or None) for i, v in enumerate(r.split(":"))) for r in sys.argv[2].split(",")]
for mode, chain, splits, ncl in runs:
    if ncl:
        os.environ["TSK_PAIR_CLUSTERS"] = ncl
    else:
        os.environ.pop("TSK_PAIR_CLUSTERS", None)
    ms = timeit(lambda: tsk.tsk_gram_probe(X, mode=mode, chain=chain, splits=splits))
    print(f"mode={mode} chain={chain} splits={splits} clusters={ncl}: {ms:.2f} ms  alg {alg / ms / 1e9:.0f} TF/s",
          flush=True)
