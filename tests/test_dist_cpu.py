"""World-size-2 gloo tests (CPU) of the column-sharded multi-GPU plumbing.

The per-rank compute is replaced by the fp64 oracle (tests only) so that the
shard arithmetic, the all-gather and the gather layout are checked on CPU; on the
GPU box the same class calls the CUDA kernels.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_09577_b200.dist import (ColumnParallelFlashNorm, gather_columns_reference, shard_bounds,
                                        shard_columns)


def test_shard_bounds():
    assert shard_bounds(28672, 8, 0) == (0, 3584)
    assert shard_bounds(28672, 8, 7) == (25088, 28672)
    assert shard_bounds(57344, 2, 1) == (28672, 57344)
    spans = [shard_bounds(6144, 4, r) for r in range(4)]
    assert spans[0][0] == 0 and spans[-1][1] == 6144
    assert all(spans[i][1] == spans[i + 1][0] for i in range(3))
    with pytest.raises(ValueError):
        shard_bounds(100, 8, 0)
    with pytest.raises(ValueError):
        shard_bounds(64, 2, 2)


def test_gather_reference_layout():
    parts = torch.arange(2 * 3 * 4).reshape(2, 3, 4)
    z = gather_columns_reference(parts)
    assert z.shape == (3, 8)
    assert torch.equal(z[:, :4], parts[0]) and torch.equal(z[:, 4:], parts[1])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_compute(a, Wt, c, eps, mode, alpha):
    from oracle import flashnorm_oracle as O
    z = O.deferred_linear(a.numpy(), Wt.numpy().T, None if c is None else c.numpy(), eps)
    return torch.from_numpy(z)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)  # same seed on every rank: replicated activations / weights
        M, K, N = 5, 32, 48
        a = torch.from_numpy(rng.standard_normal((M, K)))
        Wt = torch.from_numpy(rng.standard_normal((N, K)) / np.sqrt(K))
        c = torch.from_numpy(rng.uniform(-0.1, 0.1, N))
        layer = ColumnParallelFlashNorm.from_full(Wt, c, compute_fn=_oracle_compute,
                                                  permute_fn=gather_columns_reference)
        z_local = layer(a, gather=False)
        z_full = layer(a, gather=True)
        lo, hi = shard_bounds(N, world, rank)
        Wl, cl = shard_columns(Wt, c, world, rank)
        ok_local = torch.allclose(z_local, _oracle_compute(a, Wl, cl, 1e-5, "rmsnorm", 0.5))
        ref = _oracle_compute(a, Wt, c, 1e-5, "rmsnorm", 0.5)
        ok_full = torch.allclose(z_full, ref, rtol=1e-13, atol=1e-13)
        q.put((rank, ok_local, ok_full, tuple(z_local.shape), (lo, hi)))
    finally:
        dist.destroy_process_group()


def test_column_parallel_world2_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert [r[1] for r in res] == [True, True], res
    assert [r[2] for r in res] == [True, True], res
    assert res[0][3] == (5, 24) and res[0][4] == (0, 24) and res[1][4] == (24, 48)


def test_layernorm_exact_shards_are_row_local():
    """The deferred LayerNorm (reading c29) column-shards like the RMS path: u = 1^T W* and c* are
    per output column, mu / var are per token over the full K that every rank holds, so the
    concatenated shard outputs equal the unsharded result (no collective on the data path)."""
    from oracle import flashnorm_oracle as O
    rng = np.random.default_rng(5)
    M, K, N, world = 6, 64, 64, 4
    a = rng.standard_normal((M, K)) + rng.uniform(-3, 3, (M, 1))
    Wt = rng.standard_normal((N, K)) / np.sqrt(K)
    g, b, c = rng.uniform(0.5, 1.5, K), rng.uniform(-0.1, 0.1, K), rng.uniform(-0.1, 0.1, N)
    Ws, cs = O.fold_weights(Wt.T, g, b, c)
    full = O.layernorm_deferred(a, Ws, O.column_sums(Ws), cs, 1e-5)
    parts = []
    for rank in range(world):
        lo, hi = shard_bounds(N, world, rank)
        Wl, cl = O.fold_weights(Wt[lo:hi].T, g, b, c[lo:hi])
        parts.append(O.layernorm_deferred(a, Wl, O.column_sums(Wl), cl, 1e-5))
    np.testing.assert_allclose(np.concatenate(parts, axis=1), full, rtol=1e-12, atol=1e-12)
