"""Developer tool: dump the C3/C4 training Grams (fp64 .npy) and the full C5 spectrum to gpurun_out/
so eigensolver schedules can be studied on the CPU.  python scripts/dump_spectra.py"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402
out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out")
os.makedirs(out, exist_ok=True)
for name in ("C3", "C4"):
    c = datagen.CONFIGS[name]
    t = time.time()
    A = datagen.generate(c, "train", device="cuda")
    G, _ = tsk.sketch_gram(A)
    del A
    np.save(os.path.join(out, f"G_{name}.npy"), G.cpu().numpy())
    print(name, "gram saved", time.time() - t, flush=True)
c = datagen.CONFIGS["C5"]
G = torch.zeros(c.m, c.m, dtype=torch.float64, device="cuda")
t = time.time()
ch = 100
buf = torch.empty(ch, c.m, c.n, dtype=torch.float32, device="cuda")
for d0 in range(0, c.D_train, ch):
    datagen.generate(c, "train", d0, d0 + ch, device="cuda", out=buf)
    tsk.sketch_gram(buf, G64=G, accumulate=1)
    print("C5", d0, time.time() - t, flush=True)
w = torch.linalg.eigvalsh(G).flip(0)
np.save(os.path.join(out, "lam_C5.npy"), w.cpu().numpy())
np.save(os.path.join(out, "G_C5_f32_top.npy"), G[:1024, :1024].float().cpu().numpy())
print("C5 done", time.time() - t, w[:5].tolist(), w[95:105].tolist(), flush=True)
