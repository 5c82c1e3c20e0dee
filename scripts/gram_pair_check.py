"""Developer check of the CTA-pair Gram (gram_pair.cu): accuracy over ragged shapes against an
fp64 torch reference, then C4 timing against the 1-CTA kernel (probe mode 16).
python scripts/gram_pair_check.py [skip_timing]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


g = torch.Generator(device="cuda").manual_seed(0)
for (D, m, n) in [(3, 64, 48), (2, 8, 4), (5, 129, 36), (4, 256, 256), (3, 300, 100), (7, 1080, 1920),
                  (2, 1024, 768), (3, 200, 40), (1, 600, 4), (2, 1152, 64)]:
    X = torch.rand(D, m, n, device="cuda", generator=g) - 0.3
    Xd = X.double()
    Gref = torch.einsum("dij,dkj->ik", Xd, Xd)
    G = tsk.tsk_gram_probe(X)
    G1 = tsk.tsk_gram_probe(X, mode=16)
    e = float((G - Gref).norm() / Gref.norm())
    e1 = float((G1 - Gref).norm() / Gref.norm())
    sym = float((G - G.T).abs().max())
    print(f"D={D} m={m} n={n}: pair relF={e:.2e}  1cta relF={e1:.2e}  asym={sym:.1e}", flush=True)
    assert e < 1e-5 and sym == 0.0, (e, sym)

if len(sys.argv) < 2:
    m, n, D = 1080, 1920, 2000
    X = torch.rand(D, m, n, device="cuda")
    alg = m * (m + 1) * n * D
    for mode, name in [(0, "pair"), (16, "1cta")]:
        ms = timeit(lambda: tsk.tsk_gram_probe(X, mode=mode))
        print(f"C4 {name}: {ms:.2f} ms  alg {alg / ms / 1e9:.0f} TF/s", flush=True)
    Xs = X[:300].contiguous()
    Xd = Xs.double()
    Gref = torch.einsum("dij,dkj->ik", Xd, Xd)
    for ch in (2, 4, 8):
        e = float((tsk.tsk_gram_probe(Xs, chain=ch) - Gref).norm() / Gref.norm())
        print(f"C4[:300] pair chain={ch} relF={e:.2e}", flush=True)
print("ok")
