"""Degenerate inputs (developer check): zero / constant / rank-1 / scaled test matrices through SCW and the
two-sided SCW, zero training slices in the Gram, against the oracle."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402
from oracle import scw as oscw, tucker1, tucker2  # noqa: E402

c = datagen.CONFIGS["C2"]
A = datagen.generate(c, "train", 0, 40)
S, lam, _, _ = tsk.sketch_train(A.cuda(), c.k)
W = torch.tensor(np.linalg.qr(np.random.default_rng(0).standard_normal((c.n, 12)))[0].T.copy(), dtype=torch.float32)
m, n = c.m, c.n
cases = {
    "zero": torch.zeros(m, n),
    "constant": torch.full((m, n), 0.7),
    "rank1": torch.outer(torch.linspace(0, 1, m), torch.linspace(1, 2, n)),
    "tiny": datagen.generate(c, "test", 0, 1)[0] * 1e-12,
    "large": datagen.generate(c, "test", 0, 1)[0] * 1e12,
    "onehot": torch.zeros(m, n).index_put_((torch.tensor([5]), torch.tensor([7])), torch.tensor([3.0])),
}
for name, T in cases.items():
    T3 = T[None].contiguous()
    e = tsk.scw_error(T3.cuda(), S, c.r).cpu().numpy()
    eo = oscw.scw_errors(T3.numpy(), S.cpu().double().numpy(), c.r)
    e2 = tsk.two_sided_scw_error(T3.cuda(), S, W.cuda(), 6).cpu().numpy()
    e2o = tucker2.two_sided_scw_errors(T3.numpy(), S.cpu().double().numpy(), W.double().numpy(), 6)
    fro = float(np.linalg.norm(T3.numpy().astype(np.float64)))
    ok = np.all(np.isfinite(e)) and abs(e[0] - eo[0]) <= 1e-4 * eo[0] + 1e-6 * fro and \
        np.all(np.isfinite(e2)) and abs(e2[0] - e2o[0]) <= 1e-4 * e2o[0] + 1e-6 * fro
    print(f"{'ok ' if ok else 'BAD'} {name:9s} scw {e[0]:.6e} / {eo[0]:.6e}   two-sided {e2[0]:.6e} / {e2o[0]:.6e}")
# Gram with zero slices and a zero stack
Z = torch.zeros(3, m, n)
G, _ = tsk.sketch_gram(Z.cuda())
print("zero Gram max", float(G.abs().max()))
try:
    S0, l0, i0, s0 = tsk.sketch_topk(G, 5)
    print("topk of zero Gram: status", s0, "orth", float(torch.linalg.norm(S0.double() @ S0.double().T - torch.eye(5, dtype=torch.float64, device="cuda"))))
except Exception as ex:
    print("topk of zero Gram:", ex)
