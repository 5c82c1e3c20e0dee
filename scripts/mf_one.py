"""One matrix-free sketch call at a config, bracketed by cudaProfilerStart/Stop for
`ncu --profile-from-start off` launch lists (developer script).

  python scripts/mf_one.py [--config C4] [--oversample 4] [--q 2]
"""
import argparse, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--D", type=int, default=0)
ap.add_argument("--oversample", type=int, default=4)
ap.add_argument("--q", type=int, default=2)
a = ap.parse_args()
c = datagen.CONFIGS[a.config]
A = datagen.generate(c, "train", 0, a.D or c.D_train, device="cuda")
tsk.sketch_train_matrix_free(A, c.k, oversample=a.oversample, power_iters=a.q)
torch.cuda.synchronize()
torch.cuda.profiler.start()
tsk.sketch_train_matrix_free(A, c.k, oversample=a.oversample, power_iters=a.q)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
