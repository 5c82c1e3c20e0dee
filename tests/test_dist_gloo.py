"""Multi-rank host logic of the data-parallel path on CPU (gloo, world size 2 and 3).

The GPU kernels cannot run here, so each rank computes its shard's partial Gram with the fp64
oracle; what is under test is the product's sharding (shard_range) and its one collective
(reduce_gram): the all-reduced partial Grams must equal the single-process Gram, and every rank
must then hold the same sketch (pin P11 "shard count")."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen
from oracle import tucker1
from paper_2209_14637_b200.dist import reduce_gram, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cfg_name, k, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = datagen.CONFIGS[cfg_name]
        d0, d1 = shard_range(c.D_train, rank, world)
        A = datagen.generate(c, "train", d0, d1).numpy()
        G = torch.tensor(tucker1.mode1_gram(A) if d1 > d0 else np.zeros((c.m, c.m)))
        reduce_gram(G)
        S, lam = tucker1.top_k_eigen(G.numpy(), k)
        out[rank] = (d0, d1, G.numpy(), S)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gram_allreduce_matches_single_process(world):
    c = datagen.CONFIGS["C1"]
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), "C1", c.k, out), nprocs=world, join=True)
    ranges = sorted((out[r][0], out[r][1]) for r in range(world))
    assert ranges[0][0] == 0 and ranges[-1][1] == c.D_train
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    A = datagen.generate(c, "train").numpy()
    S_ref, _, G_ref = tucker1.tucker1_sketch(A, c.k)
    for r in range(world):
        _, _, G, S = out[r]
        np.testing.assert_allclose(G, G_ref, rtol=1e-12, atol=1e-12 * np.abs(G_ref).max())
        assert tucker1.projector_distance(S, S_ref) < 1e-9
    # every rank holds the same S (deterministic replicated eigensolver input)
    for r in range(1, world):
        np.testing.assert_array_equal(out[r][2], out[0][2])


def test_shard_range_properties():
    for D in (0, 1, 7, 2000):
        for P in (1, 2, 4, 8):
            rs = [shard_range(D, p, P) for p in range(P)]
            assert rs[0][0] == 0 and rs[-1][1] == D
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _gather_worker(rank, world, port, B, out):
    """Each rank computes the oracle SCW errors of its contiguous test shard; gather_errors returns the
    whole stream's errors in order on every rank (PAPER.md:248-252 needs all of them)."""
    from oracle import scw as oscw
    from paper_2209_14637_b200.dist import gather_errors

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = datagen.CONFIGS["C1"]
        S, _, _ = tucker1.tucker1_sketch(datagen.generate(c, "train").numpy(), c.k)
        lo, hi = shard_range(B, rank, world)
        T = datagen.generate(c, "test", lo, hi).numpy() if hi > lo else np.zeros((0, c.m, c.n), np.float32)
        e_local = torch.tensor(oscw.scw_errors(T, S, c.r) if hi > lo else np.zeros(0))
        out[rank] = gather_errors(e_local, B).numpy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,B", [(2, 10), (3, 10), (3, 2)])
def test_gather_errors_matches_single_process(world, B):
    """Sharded test stream (ragged shards, and an empty one when B < world) -> gathered errors equal the
    single-process errors bit for bit, on every rank, and give the same paper test error."""
    from oracle import scw as oscw

    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_gather_worker, args=(world, _free_port(), B, out), nprocs=world, join=True)
    c = datagen.CONFIGS["C1"]
    S, _, _ = tucker1.tucker1_sketch(datagen.generate(c, "train").numpy(), c.k)
    T = datagen.generate(c, "test", 0, B).numpy()
    e_ref = oscw.scw_errors(T, S, c.r)
    eopt = np.array([oscw.best_rank_r_error(a, c.r) for a in T])
    for r in range(world):
        np.testing.assert_array_equal(out[r], e_ref)
        assert oscw.test_error(out[r], eopt) == oscw.test_error(e_ref, eopt)


def _train_worker(rank, world, port, D, out):
    """dist.train's own control flow with fp64 stand-ins for the GPU calls: a rank whose shard is empty
    (D < world) must still join the Gram all-reduce instead of raising and leaving its peers blocked."""
    from paper_2209_14637_b200.dist import train

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = datagen.CONFIGS["C1"]
        lo, hi = shard_range(D, rank, world)
        A = datagen.generate(c, "train", lo, hi) if hi > lo else torch.zeros((0, c.m, c.n))

        def gram_fn(A_local, G64=None, opts=None):
            return torch.tensor(tucker1.mode1_gram(A_local.numpy())), None

        def topk_fn(G64, k, opts=None):
            S, lam = tucker1.top_k_eigen(G64.numpy(), k)

            class _Info:
                gram_splits = gram_tiles = 0
            return torch.tensor(S), torch.tensor(lam[:k]), _Info(), 0

        S, lam, info, st = train(A, c.k, gram_fn=gram_fn, topk_fn=topk_fn)
        out[rank] = S.numpy()
    finally:
        dist.destroy_process_group()


def test_train_with_an_empty_shard():
    world, D = 3, 2
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_train_worker, args=(world, _free_port(), D, out), nprocs=world, join=True)
    c = datagen.CONFIGS["C1"]
    S_ref, _, _ = tucker1.tucker1_sketch(datagen.generate(c, "train", 0, D).numpy(), c.k)
    for r in range(world):
        assert tucker1.projector_distance(out[r], S_ref) < 1e-9
