"""Randomised sweep of the API variants (developer check): host vs device pointers (bitwise), streamed
accumulate vs one call, G32 output, factors vs errors.  python scripts/random_sweep3.py [n_cases] [seed]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402

ncase = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
for t in range(ncase):
    m = int(rng.integers(2, 600)); n = int(rng.integers(1, 150)) * 4; D = int(rng.integers(2, 30))
    A = torch.from_numpy(rng.random((D, m, n), dtype=np.float32) - 0.3)
    msg, ok = [], True
    Gd, _ = tsk.sketch_gram(A.cuda())
    Gh, _ = tsk.sketch_gram(A)                     # host input (pageable), streamed by the library
    Gp, _ = tsk.sketch_gram(A.pin_memory())        # pinned
    eq = torch.equal(Gd.cpu(), Gh.cpu()) and torch.equal(Gd.cpu(), Gp.cpu()); ok &= eq; msg.append(f"host={'=' if eq else 'DIFF'}")
    h = int(rng.integers(1, D))
    Ga, _ = tsk.sketch_gram(A[:h].cuda())
    tsk.sketch_gram(A[h:].cuda(), G64=Ga, accumulate=True)
    e = float((Ga - Gd).norm() / Gd.norm()); ok &= e <= 1e-6; msg.append(f"acc={e:.1e}")
    G32 = torch.empty(m, m, dtype=torch.float32, device="cuda")
    G64b, _ = tsk.sketch_gram(A.cuda(), G32=G32)
    e = float((G32.double() - G64b).abs().max() / G64b.abs().max()); ok &= e <= 1e-6; msg.append(f"g32={e:.1e}")
    k = int(rng.integers(1, min(m, 40) + 1)); r = int(rng.integers(1, min(k, n, 64) + 1))
    S, lam, info, st = tsk.sketch_train(A.cuda(), k)
    T = torch.from_numpy(rng.random((4, m, n), dtype=np.float32) - 0.3)
    ed = tsk.scw_error(T.cuda(), S, r).cpu()
    eh = tsk.scw_error(T, S.cpu(), r)
    eq = torch.equal(ed, eh.cpu()); ok &= eq; msg.append(f"scw_host={'=' if eq else 'DIFF'}")
    L, R, sg = tsk.sketch_apply_scw(T.cuda(), S, r)
    ef = torch.linalg.norm((T.cuda().double() - torch.bmm(L.double(), R.double().transpose(1, 2))).reshape(4, -1), dim=1).cpu()
    e = float(((ef - ed).abs() / ed).max()); ok &= e <= 1e-5; msg.append(f"fac/err={e:.1e}")
    bad += not ok
    print(("ok  " if ok else "BAD ") + f"m={m} n={n} D={D} h={h} k={k} r={r} " + " ".join(msg), flush=True)
print("failures:", bad)
