"""Two contexts used from two host threads concurrently (the ABI's threading promise, developer check):
results must equal the serial ones bit for bit."""
import os, sys, threading
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402

c = datagen.CONFIGS["C3"]
A = [datagen.generate(c, "train", 40 * i, 40 * i + 40, device="cuda") for i in range(2)]
T = datagen.generate(c, "test", 0, 20, device="cuda")
ref = []
for i in range(2):
    S, lam, _, _ = tsk.sketch_train(A[i], c.k)
    ref.append((S.clone(), lam.clone(), tsk.scw_error(T, S, c.r).clone()))
torch.cuda.synchronize()
out = [None, None]

def work(i):
    with torch.cuda.stream(torch.cuda.Stream()):
        ctx = tsk.Context(0)
        for _ in range(3):
            S, lam, _, _ = tsk.sketch_train(A[i], c.k, ctx=ctx)
            e = tsk.scw_error(T, S, c.r, ctx=ctx)
        torch.cuda.current_stream().synchronize()
        out[i] = (S, lam, e)
        ctx.close()

th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
[t.start() for t in th]
[t.join() for t in th]
for i in range(2):
    same = all(torch.equal(a, b) for a, b in zip(out[i], ref[i]))
    print("thread", i, "bitwise equal to serial:", same)
