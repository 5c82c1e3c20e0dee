"""The seeded input generator (no method arithmetic).  CPU only."""
import numpy as np
import pytest
import torch

import datagen


def test_configs_match_baseline():
    c = datagen.CONFIGS
    assert (c["C1"].m, c["C1"].n, c["C1"].D_train, c["C1"].D_test, c["C1"].k, c["C1"].r) == (64, 48, 20, 10, 10, 5)
    assert (c["C2"].m, c["C2"].n, c["C2"].D_train, c["C2"].D_test, c["C2"].k, c["C2"].r) == (256, 256, 200, 100, 20, 10)
    assert (c["C3"].m, c["C3"].n, c["C3"].D_train, c["C3"].D_test, c["C3"].k, c["C3"].r) == (1024, 768, 400, 200, 40, 20)
    assert (c["C4"].m, c["C4"].n, c["C4"].D_train, c["C4"].D_test, c["C4"].k, c["C4"].r) == (1080, 1920, 2000, 500, 60, 30)
    assert (c["C5"].m, c["C5"].n, c["C5"].D_train, c["C5"].D_test, c["C5"].k, c["C5"].r) == (4096, 4096, 2000, 256, 100, 50)


def test_deterministic_and_shardable():
    a = datagen.generate("C1", "train")
    b = datagen.generate("C1", "train")
    assert a.dtype == torch.float32 and a.shape == (20, 64, 48) and a.is_contiguous()
    assert torch.equal(a, b)
    part = datagen.generate("C1", "train", 7, 13)
    assert torch.equal(part, a[7:13])
    t = datagen.generate("C1", "test")
    assert t.shape == (10, 64, 48)
    assert not torch.equal(t[0], a[0])
    assert not torch.equal(datagen.generate("C1", "train", seed=1)[0], a[0])


def test_frame_like_in_unit_interval():
    c = datagen.CONFIGS["C3"].replace(m=96, n=64, p=10, D_train=3, D_test=1)
    a = datagen.generate(c, "train")
    assert float(a.min()) >= 0.0 and float(a.max()) <= 1.0
    assert 0.4 < float(a.mean()) < 0.6


def test_lowrank_variant_has_exact_rank():
    c = datagen.lowrank("C1", rank=5)
    a = datagen.generate(c, "test").double().numpy()
    for A in a:
        s = np.linalg.svd(A, compute_uv=False)
        assert s[5] <= 1e-6 * s[0]


def test_identical_variant():
    c = datagen.identical("C1", D_train=4)
    a = datagen.generate(c, "train")
    for d in range(1, 4):
        assert torch.equal(a[d], a[0])


def test_bad_range():
    with pytest.raises(ValueError):
        datagen.generate("C1", "train", 0, 21)


def test_random_sign_sketch_pattern():
    """one nonzero per column, values +-1, deterministic under the seed; k = 1 is
    a single row of +-1."""
    S = datagen.random_sign_sketch(7, 50, seed=3)
    assert S.shape == (7, 50)
    nz = (S != 0).sum(dim=0)
    assert torch.all(nz == 1)
    assert torch.all(S.abs().sum(dim=0) == 1)
    assert torch.equal(S, datagen.random_sign_sketch(7, 50, seed=3))
    assert not torch.equal(S, datagen.random_sign_sketch(7, 50, seed=4))
    S1 = datagen.random_sign_sketch(1, 9, seed=0)
    assert torch.all(S1.abs() == 1)


def test_random_gaussian_sketch_moments():
    """determinism; mean ~ 0 within 5 standard errors at k*m = 1e4; E||Sx||^2 ~ ||x||^2
    within 20% (JL expectation) for unit x averaged over 100 seeds."""
    S = datagen.random_gaussian_sketch(20, 500, seed=1)
    assert torch.equal(S, datagen.random_gaussian_sketch(20, 500, seed=1))
    se = (1.0 / 20) ** 0.5 / (S.numel() ** 0.5)
    assert abs(float(S.double().mean())) <= 5 * se
    x = torch.randn(500, dtype=torch.float64, generator=torch.Generator().manual_seed(0))
    x /= x.norm()
    vals = [float((datagen.random_gaussian_sketch(20, 500, seed=s).double() @ x).pow(2).sum()) for s in range(100)]
    assert abs(sum(vals) / len(vals) - 1.0) <= 0.2
