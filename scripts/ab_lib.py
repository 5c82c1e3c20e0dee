"""A/B timing of two builds of libtsketch.so in one process (developer tool):
python scripts/ab_lib.py A.so B.so [rounds] -- times the C4 Gram (tsk_gram_probe, datagen stream) with
each library in alternation (ctypes loads both; contexts are per library)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402

libs = sys.argv[1:3]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 4
c = datagen.CONFIGS["C4"]
A = datagen.generate(c, "train", device="cuda")
loaded = {}
for p in libs:
    tsk._lib = None
    tsk.LIB_PATH = os.path.abspath(p)
    tsk._ctx_cache.clear()
    loaded[p] = (tsk.lib(), tsk.context(0))
for r in range(rounds):
    for p in libs:
        tsk._lib, ctx = loaded[p]
        tsk._ctx_cache[0] = ctx
        tsk.tsk_gram_probe(A, ctx=ctx)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            tsk.tsk_gram_probe(A, ctx=ctx)
        e1.record()
        torch.cuda.synchronize()
        print(f"{os.path.basename(p)} round {r}: {e0.elapsed_time(e1) / 3:.2f} ms", flush=True)
