"""Time the matrix-free sketch (randomized block Krylov) against the exact sketch
(Gram + eigensolver) on a config's training stream; CUDA events on the current stream.

  python scripts/mf_time.py [--config C4] [--D 2000] [--oversample 4] [--q 2]
"""
import argparse, json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); out = fn(); b.record(); torch.cuda.synchronize()
        t = a.elapsed_time(b)
        best = t if best is None else min(best, t)
    return best, out


ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--D", type=int, default=0)
ap.add_argument("--oversample", type=int, default=4)
ap.add_argument("--q", type=str, default="1,2")
ap.add_argument("--subspace", action="store_true")
a = ap.parse_args()
c = datagen.CONFIGS[a.config]
D = a.D or c.D_train
A = datagen.generate(c, "train", 0, D, device="cuda")
T = datagen.generate(c, "test", 0, 32, device="cuda")
t0, (S0, lam0, _, _) = timed(lambda: tsk.sketch_train(A, c.k))
e0 = tsk.scw_error(T, S0, c.r)
print(json.dumps({"config": a.config, "D": D, "method": "exact (Gram + eig)", "ms": round(t0, 2),
                  "kyfan": float(lam0.sum()), "mean_scw_err": float(e0.mean())}), flush=True)
for q in [int(x) for x in a.q.split(",")]:
    t1, (S, lam, info, st) = timed(lambda: tsk.sketch_train_matrix_free(A, c.k, oversample=a.oversample,
                                                                        power_iters=q, subspace=a.subspace))
    e1 = tsk.scw_error(T, S, c.r)
    print(json.dumps({"config": a.config, "D": D, "method": "matrix-free", "q": q, "info": info, "ms": round(t1, 2),
                      "kyfan_rel_deficit": float(1 - lam.sum() / lam0.sum()),
                      "mean_scw_err_rel_excess": float((e1 - e0).mean() / e0.mean())}), flush=True)
