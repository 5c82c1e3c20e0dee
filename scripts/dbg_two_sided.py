"""Debug: two-sided SCW per-matrix errors vs the oracle for random orthonormal S, W (developer check)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_2209_14637_b200 as tsk
from oracle import tucker2
def orth_rows(rng, k, m):
    q, _ = np.linalg.qr(rng.standard_normal((m, k)))
    return q.T.copy()
for (m, n, k, l, r, B) in [(188, 204, 18, 6, 5, 3), (188, 204, 18, 8, 5, 3), (192, 204, 18, 6, 5, 3), (188, 256, 18, 6, 5, 3),
                           (188, 204, 16, 6, 5, 3), (188, 204, 18, 6, 6, 3), (64, 48, 10, 6, 5, 3), (128, 128, 18, 6, 5, 3)]:
    rng = np.random.default_rng(0)
    T = torch.from_numpy(rng.random((B, m, n), dtype=np.float32) - 0.3)
    S = orth_rows(rng, k, m); W = orth_rows(rng, l, n)
    e = tsk.two_sided_scw_error(T.cuda(), torch.tensor(S, dtype=torch.float32).cuda(), torch.tensor(W, dtype=torch.float32).cuda(), r).cpu().numpy()
    eo = tucker2.two_sided_scw_errors(T.numpy(), S.astype(np.float32).astype(np.float64), W.astype(np.float32).astype(np.float64), r)
    print((m, n, k, l, r, B), np.round(np.abs(e - eo) / eo, 8))
# per-matrix vs batched, and the one-sided SCW at the failing shape
m, n, k, l, r, B = 188, 204, 18, 6, 5, 3
rng = np.random.default_rng(0)
T = torch.from_numpy(rng.random((B, m, n), dtype=np.float32) - 0.3)
S = torch.tensor(orth_rows(rng, k, m), dtype=torch.float32).cuda(); W = torch.tensor(orth_rows(rng, l, n), dtype=torch.float32).cuda()
eb = tsk.two_sided_scw_error(T.cuda(), S, W, r).cpu().numpy()
ei = np.array([float(tsk.two_sided_scw_error(T[i:i + 1].cuda(), S, W, r).cpu()[0]) for i in range(B)])
print("batched", eb, "single", ei)
L, R, sg = tsk.sketch_apply_two_sided_scw(T.cuda(), S, W, r)
Lb = [tsk.sketch_apply_two_sided_scw(T[i:i + 1].cuda(), S, W, r) for i in range(B)]
for i in range(B):
    print(i, "L diff", float((L[i] - Lb[i][0][0]).abs().max()), "R diff", float((R[i] - Lb[i][1][0]).abs().max()), "sig", sg[i].cpu().numpy(), Lb[i][2][0].cpu().numpy())
from oracle import scw as oscw
e1 = tsk.scw_error(T.cuda(), S, r).cpu().numpy(); e1o = oscw.scw_errors(T.numpy(), S.cpu().double().numpy(), r)
print("one-sided rel", np.abs(e1 - e1o) / e1o)
A3 = T.numpy().astype(np.float64)
Sd, Wd = S.cpu().double().numpy(), W.cpu().double().numpy()
for i in range(B):
    Lo, so, Ro = tucker2.two_sided_scw_factors(A3[i], Sd, Wd, r)
    eo = np.linalg.norm(A3[i] - Lo @ Ro.T)
    eg = np.linalg.norm(A3[i] - L[i].cpu().double().numpy() @ R[i].cpu().double().numpy().T)
    print(i, "oracle sigma", np.round(so, 4), "gpu sigma", np.round(sg[i].cpu().numpy(), 4), "err oracle", eo, "gpu(LR)", eg, "gpu err", eb[i])
    Q, _ = np.linalg.qr(A3[i].T @ Sd.T); P, _ = np.linalg.qr(A3[i] @ Wd.T)
    print("   svals of A W^T", np.round(np.linalg.svd(A3[i] @ Wd.T, compute_uv=False), 4))
