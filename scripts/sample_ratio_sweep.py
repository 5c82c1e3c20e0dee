"""Sample-ratio sweep (Fig. 2): test error of the tensor-based
and the two-sided tensor-based algorithms when the training set is a fraction
sample_ratio = D_train / (D_train + D_test) of the stream (the paper uses 2 %, 20 %, 80 %), on the
synthetic stand-in streams (the HSI/Logo/MRI datasets are not available).

Everything runs through the GPU C ABI; e_opt = ||A - [A]_r||_F (the metric's denominator) comes
from torch's SVD of each test matrix (an evaluation step, not part of the method).

  python scripts/sample_ratio_sweep.py [--config C2] [--ratios 0.02,0.2,0.8] [--seed 0]

Prints one JSON line per ratio and a final line with err(80 %) / err(2 %), the factor the paper reports
(tensor-based 0.952 / 0.917 / 0.684, two-sided 0.873 / 0.789 / 0.606 on HSI / Logo / MRI; context only).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2209_14637_b200 as tsk  # noqa: E402


def test_error(err: torch.Tensor, eopt: torch.Tensor) -> float:
    """Mean of (e - e_opt) / e_opt over the test set; e_opt = 0 terms excluded (reading c13)."""
    keep = eopt > 0
    return float(((err[keep] - eopt[keep]) / eopt[keep]).mean())


def sweep(cfg: str = "C2", ratios=(0.02, 0.2, 0.8), seed: int = 0, l: int | None = None):
    c = datagen.CONFIGS[cfg]
    l = l or c.k
    T = datagen.generate(c, "test", seed=seed).cuda()
    eopt = torch.stack([torch.linalg.svdvals(t.double())[c.r:].pow(2).sum().sqrt() for t in T])
    out = []
    for ratio in ratios:
        ntr = max(1, round(ratio / (1.0 - ratio) * c.D_test))
        cc = c.replace(D_train=max(c.D_train, ntr))
        A = datagen.generate(cc, "train", 0, ntr, seed=seed).cuda()
        S, _, _, _ = tsk.sketch_train(A, c.k)
        e1 = tsk.scw_error(T, S, c.r)
        S2, W2, info, _ = tsk.sketch_train_two_sided(A, c.k, l, max_sweeps=5)
        e2 = tsk.two_sided_scw_error(T, S2, W2, c.r)
        out.append({"config": cfg, "sample_ratio": ratio, "D_train": ntr, "D_test": c.D_test, "k": c.k, "l": l,
                    "r": c.r, "test_error_tensor_based": test_error(e1.cpu(), eopt.cpu()),
                    "test_error_two_sided": test_error(e2.cpu(), eopt.cpu()), "hooi_sweeps": info["sweeps"]})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--ratios", default="0.02,0.2,0.8")
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    rows = sweep(args.config, tuple(float(x) for x in args.ratios.split(",")), args.seed)
    for row in rows:
        print(json.dumps(row), flush=True)
    print(json.dumps({"factor_tensor_based": rows[-1]["test_error_tensor_based"] / rows[0]["test_error_tensor_based"],
                      "factor_two_sided": rows[-1]["test_error_two_sided"] / rows[0]["test_error_two_sided"],
                      "paper_context": {"tensor_based": [0.952, 0.917, 0.684], "two_sided": [0.873, 0.789, 0.606]}}))


if __name__ == "__main__":
    main()
