"""Quick numerics check of every stage on a B200 (developer script; the gated tests live in tests/)."""
import sys
import time
import traceback

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402
from oracle import scw as oscw, tucker1  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def section(name, fn):
    print(f"=== {name}", flush=True)
    t = time.time()
    try:
        fn()
    except Exception:
        traceback.print_exc()
    print(f"    ({time.time() - t:.1f}s)", flush=True)


def gram_case(D, m, n, seed=0, **opts):
    g = torch.Generator().manual_seed(seed)
    A = torch.rand(D, m, n, generator=g, dtype=torch.float32)
    Gd, info = tsk.sketch_gram(A.cuda(), opts=opts or None)
    torch.cuda.synchronize()
    Go = tucker1.mode1_gram(A.numpy())
    Gg = Gd.cpu().numpy()
    print(f"  gram D={D} m={m} n={n} opts={opts}: relF={rel(Gg, Go):.3e} sym={np.abs(Gg - Gg.T).max():.1e} "
          f"splits={info.gram_splits} tiles={info.gram_tiles}", flush=True)


def main():
    print(torch.cuda.get_device_name(), flush=True)
    section("gram tiny", lambda: gram_case(2, 64, 32))
    section("gram C1-shape", lambda: gram_case(20, 64, 48))
    section("gram ragged", lambda: gram_case(7, 300, 100))
    section("gram 256", lambda: gram_case(10, 256, 256))
    for ch in (1, 4, 16, 64):
        section(f"gram chain={ch}", lambda ch=ch: gram_case(8, 256, 1024, gemm_chain=ch))
    section("gram C4-shape", lambda: gram_case(4, 1080, 1920))

    def topk_c1():
        A = datagen.generate("C1", "train")
        S, lam, info, st = tsk.sketch_train(A.cuda(), 10)
        torch.cuda.synchronize()
        So, lamo, Go = tucker1.tucker1_sketch(A.numpy(), 10)
        print(f"  C1 projector={tucker1.projector_distance(S.cpu().double().numpy(), So):.3e} "
              f"lam rel={rel(lam.cpu().numpy(), lamo[:10]):.3e} status={st} info={info.as_dict()}")
        print(f"  gap={tucker1.eigengap(lamo, 10):.4f}")
    section("train C1 (dense)", topk_c1)

    def topk_sub():
        c = datagen.planted("C3", gap=1.2, D_train=30).replace(m=512, n=256)
        A = datagen.generate(c, "train")
        t = time.time()
        S, lam, info, st = tsk.sketch_train(A.cuda(), c.k)
        torch.cuda.synchronize()
        print(f"  time {time.time()-t:.3f}s")
        So, lamo, Go = tucker1.tucker1_sketch(A.numpy(), c.k)
        Sg = S.cpu().double().numpy()
        print(f"  planted 512 projector={tucker1.projector_distance(Sg, So):.3e} gap={tucker1.eigengap(lamo, c.k):.3f} "
              f"kyfan_def={(lamo[:c.k].sum() - tucker1.kyfan_energy(Go, Sg)) / lamo[:c.k].sum():.3e} "
              f"status={st} info={info.as_dict()}")
    section("train subspace planted", topk_sub)

    def scw_c1():
        A = datagen.generate("C1", "train")
        T = datagen.generate("C1", "test")
        So, _, _ = tucker1.tucker1_sketch(A.numpy(), 10)
        S32 = torch.tensor(So, dtype=torch.float32)
        err = tsk.scw_error(T.cuda(), S32.cuda(), 5).cpu().numpy()
        eo = oscw.scw_errors(T.numpy(), S32.double().numpy(), 5)
        print(f"  C1 scw err rel max={np.max(np.abs(err - eo) / eo):.3e}  e={err[:3]} eo={eo[:3]}")
        L, R, sig = tsk.sketch_apply_scw(T.cuda(), S32.cuda(), 5)
        Lo, so, Ro = oscw.scw_factors(T[0].numpy(), S32.double().numpy(), 5)
        Ah = (L[0].double() @ R[0].double().T).cpu().numpy()
        print(f"  A_hat rel={rel(Ah, Lo @ Ro.T):.3e} sigma rel={rel(sig[0].cpu().numpy(), so):.3e}")
    section("scw C1", scw_c1)

    def e2e_c2():
        c = datagen.CONFIGS["C2"]
        A = datagen.generate(c, "train")
        T = datagen.generate(c, "test")
        S, lam, info, st = tsk.sketch_train(A.cuda(), c.k)
        So, lamo, Go = tucker1.tucker1_sketch(A.numpy(), c.k)
        Sg = S.cpu().double().numpy()
        print(f"  C2 kyfan_def={(lamo[:c.k].sum() - tucker1.kyfan_energy(Go, Sg)) / lamo[:c.k].sum():.3e} "
              f"info={info.as_dict()} st={st}")
        err = tsk.scw_error(T.cuda(), S.cuda(), c.r).cpu().numpy()
        eo = oscw.scw_errors(T.numpy(), Sg.astype(np.float32).astype(np.float64), c.r)
        print(f"  C2 scw rel max={np.max(np.abs(err - eo) / eo):.3e}")
        # host-pointer path
        err_h = tsk.scw_error(T, S.cpu(), c.r).numpy()
        print(f"  host path max diff={np.max(np.abs(err_h - err)):.3e}")
    section("C2 end-to-end", e2e_c2)


if __name__ == "__main__":
    main()
