"""Developer timing probe: Gram kernel vs chain length, eigensolver and SCW at C4 (B200)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402


def timeit(fn, reps=3, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
    c = datagen.CONFIGS[cfg]
    t = time.time()
    A = datagen.generate(c, "train", device="cuda")
    T = datagen.generate(c, "test", device="cuda")
    torch.cuda.synchronize()
    print(f"gen {cfg} {time.time() - t:.1f}s  A={tuple(A.shape)}", flush=True)
    m, n, D = c.m, c.n, c.D_train
    alg = m * (m + 1) * n * D
    G64 = torch.empty(m, m, dtype=torch.float64, device="cuda")
    Gref = None
    for ch in (1, 2, 4, 8):
        ms = timeit(lambda: tsk.sketch_gram(A, G64=G64, opts={"gemm_chain": ch}))
        g = G64.clone()
        if Gref is None:
            # fp64 reference on a subset of the stream (cuBLAS dgemm, dev check only)
            Ad = A[:200].double()
            Gref = torch.einsum("dij,dkj->ik", Ad, Ad)
        Gs, _ = tsk.sketch_gram(A[:200].contiguous(), opts={"gemm_chain": ch})
        err = (Gs - Gref).norm() / Gref.norm()
        print(f"chain={ch}: {ms:.2f} ms  alg {alg / ms / 1e9:.1f} TFLOP/s  issued(x3) {3 * alg / ms / 1e9:.1f}  "
              f"relF(200)={err:.3e}", flush=True)
    t0 = time.time()
    S, lam, info, st = tsk.sketch_topk(G64, c.k)
    torch.cuda.synchronize()
    print(f"topk first: {1e3 * (time.time() - t0):.1f} ms  info={info.as_dict()} st={st}", flush=True)
    ms = timeit(lambda: tsk.sketch_topk(G64, c.k), reps=2)
    print(f"topk: {ms:.2f} ms", flush=True)
    ms = timeit(lambda: tsk.scw_error(T, S, c.r), reps=2)
    print(f"scw_error {T.shape[0]} mats: {ms:.2f} ms  ({T.shape[0] / ms * 1e3:.0f} mats/s)", flush=True)
    ms = timeit(lambda: tsk.sketch_train(A, c.k), reps=2)
    print(f"sketch_train: {ms:.2f} ms  -> {D / ms * 1e3:.0f} training matrices/s", flush=True)


if __name__ == "__main__":
    main()
