"""Streaming sketch: the Gram of a stream accumulates chunk by chunk
(G_{t+1} = G_t + sum_{d in chunk} A_d A_d^T; PAPER.md:306 notes the whole training tensor need not be
loaded at once, P:340 names pass-efficient/streaming variants as future work) and the top-k solve is
warm-started from the previous sketch.  Parity: the streamed G equals the one-shot Gram (<= 1e-5), the
warm-started S has the same Ky Fan energy as the exact top-k (deficit <= 1e-6) and needs no more
iterations than a cold start."""
import numpy as np
import pytest
import torch

import datagen
import paper_2209_14637_b200 as tsk
from oracle import tucker1

pytestmark = pytest.mark.gpu


def test_streamed_gram_and_warm_start():
    c = datagen.CONFIGS["C3"]
    A = datagen.generate(c, "train", 0, 24).cuda()
    G = tsk.sketch_gram(A[:12])[0]
    S1, _, info1, _ = tsk.sketch_topk(G, c.k)
    tsk.sketch_gram(A[12:], G64=G, accumulate=True)          # stream the next chunk in
    Go = tucker1.mode1_gram(A.cpu().numpy())
    assert float(np.linalg.norm(G.cpu().numpy() - Go) / np.linalg.norm(Go)) <= 1e-5
    S_cold, _, ic, _ = tsk.sketch_topk(G, c.k)
    S_warm, _, iw, _ = tsk.sketch_topk(G, c.k, opts={"init_S": S1})
    lam = np.linalg.eigvalsh(Go)[::-1]
    for S in (S_cold, S_warm):
        Sg = S.cpu().double().numpy()
        deficit = (lam[:c.k].sum() - tucker1.kyfan_energy(Go, Sg)) / lam[:c.k].sum()
        assert abs(deficit) <= 1e-6
        assert np.linalg.norm(Sg @ Sg.T - np.eye(c.k)) <= 1e-5
    assert iw.iters <= ic.iters, (iw.iters, ic.iters)
