"""Diagnostic: per-phase cycles of trd_kernel (build with -DTSK_TRD_PROF; copy over libtsketch.so first).
python scripts/trd_prof.py [p ...]"""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402
L = tsk.lib()
for p in [int(a) for a in sys.argv[1:]] or [48, 76, 96, 128]:
    rng = np.random.default_rng(0)
    Q = np.linalg.qr(rng.standard_normal((p, p)))[0]
    H = torch.tensor((Q * np.exp(rng.uniform(-8, 8, p))) @ Q.T, device="cuda")
    for _ in range(3):
        tsk.tsk_syev_probe(H)
    torch.cuda.synchronize()
    out = (ctypes.c_longlong * 4)()
    L.tsk_trd_prof_read(out)
    steps = p - 2
    print(f"p={p}: per step cycles  phase1(warp0 Householder + barrier) {out[0] / steps:.0f}  "
          f"phase2(fused pass + barrier) {out[1] / steps:.0f}  phase3(w update + barrier) {out[2] / steps:.0f}  "
          f"total {(out[0] + out[1] + out[2]) / steps:.0f}")
