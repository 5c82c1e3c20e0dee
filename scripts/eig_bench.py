"""Eigensolver (sketch_topk) on the C3 / C4 / C5 training Grams: time, products, Ky Fan deficit against
fp64 eigvalsh of the same Gram (total and excluding a locked dominant pair).  TSK_EIG_TRACE=1 for the
per-iteration lines; PROFILE=1 brackets the last repetition with cudaProfilerStart/Stop (ncu
--profile-from-start off).  python scripts/eig_bench.py [C3 C4 C5]"""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402

names = sys.argv[1:] or ["C3", "C4", "C5"]
opts = {"oversample": int(os.environ["OVERSAMPLE"])} if os.environ.get("OVERSAMPLE") else None
for name in names:
    c = datagen.CONFIGS[name]
    G = torch.zeros(c.m, c.m, dtype=torch.float64, device="cuda")
    ch = 200 if c.m < 2048 else 50
    buf = torch.empty(ch, c.m, c.n, dtype=torch.float32, device="cuda")
    for d0 in range(0, c.D_train, ch):
        d1 = min(c.D_train, d0 + ch)
        datagen.generate(c, "train", d0, d1, device="cuda", out=buf[: d1 - d0])
        tsk.sketch_gram(buf[: d1 - d0], G64=G, accumulate=d0 > 0)
    del buf
    torch.cuda.empty_cache()
    w = torch.linalg.eigvalsh(G).flip(0)
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        prof = rep == 2 and os.environ.get("PROFILE")
        if prof:
            torch.cuda.profiler.start()
        e0.record()
        S, lam, info, st = tsk.sketch_topk(G, c.k, opts=opts)
        e1.record()
        torch.cuda.synchronize()
        if prof:
            torch.cuda.profiler.stop()
        Sd = S.double()
        kf = torch.trace(Sd @ G @ Sd.T).item()
        tot = w[: c.k].sum().item()
        print(f"{name} topk {e0.elapsed_time(e1):.3f} ms products={info.iters} max_resid={info.max_resid:.2e} "
              f"status={st} kyfan deficit={(tot - kf) / tot:.2e} excl. top={(tot - kf) / w[1:c.k].sum().item():.2e} "
              f"orth={torch.linalg.norm(Sd @ Sd.T - torch.eye(c.k, device='cuda', dtype=torch.float64)).item():.1e}",
              flush=True)
