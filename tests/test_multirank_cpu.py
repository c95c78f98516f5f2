"""N>1 host logic on CPU (gloo, world size 2): row sharding, the NCCL-id
broadcast of the binding, and the data-parallel decomposition of one
G-evaluation -- per-rank partials [S | N | E | changed] summed across ranks
equal the full-data update, energy and convergence count (Eq. 1, Eq. 4,
PAPER.md:122).  The partials here are computed with the oracle's primitives;
the GPU path's own partials are checked the same way in test_gpu_multihandle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1805_10638_b200 import synthetic


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partials(X, C, labels, prev):
    K, d = C.shape
    S = np.zeros((K, d))
    np.add.at(S, labels, X.astype(np.float64))
    N = np.bincount(labels, minlength=K).astype(np.float64)
    E = oracle.energy(X, C, labels) if len(X) else 0.0
    ch = float((labels != prev).sum())
    return np.concatenate([S.ravel(), N, [E, ch]])


def _worker(rank, world, port, cfg, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, C0, c = synthetic.make(cfg, N=6001)
        lo, hi = synthetic.shard_bounds(c.N, rank, world)
        C = C0.astype(np.float64) + 0.01
        prev = oracle.assign(X, C0.astype(np.float64))
        lab = oracle.assign(X[lo:hi], C)
        part = torch.from_numpy(_partials(X[lo:hi], C, lab, prev[lo:hi]))
        dist.all_reduce(part)
        # the binding's id broadcast (gloo path); the id itself needs only the NCCL library
        from paper_1805_10638_b200 import aakm
        uid = aakm.broadcast_uid(rank)
        ids = [torch.zeros(128, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(ids, torch.tensor(list(uid), dtype=torch.uint8))
        if rank == 0:
            np.save(out + ".npy", part.numpy())
            np.save(out + "_ids.npy", torch.stack(ids).numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_gloo_two_rank_decomposition(tmp_path, cfg):
    out = str(tmp_path / "part")
    mp.spawn(_worker, args=(2, _free_port(), cfg, out), nprocs=2, join=True)
    got = np.load(out + ".npy")
    ids = np.load(out + "_ids.npy")
    assert (ids[0] == ids[1]).all() and ids[0].any()
    X, C0, c = synthetic.make(cfg, N=6001)
    C = C0.astype(np.float64) + 0.01
    prev = oracle.assign(X, C0.astype(np.float64))
    lab = oracle.assign(X, C)
    ref = _partials(X, C, lab, prev)
    K, d = C.shape
    np.testing.assert_allclose(got[:K * d], ref[:K * d], rtol=1e-12, atol=1e-9)
    np.testing.assert_array_equal(got[K * d:K * d + K], ref[K * d:K * d + K])
    assert abs(got[-2] - ref[-2]) <= 1e-12 * ref[-2]
    assert got[-1] == ref[-1]
    # the combined partials give the full update step (Eq. 4)
    G_ref, _ = oracle.update(X, lab, C)
    N = got[K * d:K * d + K]
    G = np.where(N[:, None] > 0, got[:K * d].reshape(K, d) / np.maximum(N, 1)[:, None], C)
    np.testing.assert_allclose(G, G_ref, rtol=1e-12, atol=1e-12)


def test_make_shard_matches_make():
    # each rank draws only its rows (bench.py at N > 1); bytes equal make()'s slice
    from paper_1805_10638_b200 import synthetic as S
    for cfg, N, K in (("c3", 70_000, 32), ("c5", 1_200_000, 64)):
        X, C0, _ = S.make(cfg, N=N, K=K)
        for world in (1, 2, 3):
            parts = []
            for r in range(world):
                Xs, C0s, _ = S.make_shard(cfg, r, world, N=N, K=K)
                assert np.array_equal(C0s, C0)
                parts.append(Xs)
            assert np.array_equal(np.concatenate(parts), X)


def _bench_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        # each rank's own duration; the job's time is the slowest rank's
        t = bench.max_over_ranks(1.5 + rank, world, device="cpu")
        # every rank draws only its rows; the shards tile the config
        X, C0, c = synthetic.make_shard("c1", rank, world)
        lo, hi = synthetic.shard_bounds(c.N, rank, world)
        sizes = torch.tensor([hi - lo, X.shape[0]], dtype=torch.int64)
        dist.all_reduce(sizes)
        if rank == 0:
            np.save(out + ".npy", np.array([t, sizes[0].item(), sizes[1].item(), c.N]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_bench_rank_plumbing(tmp_path, world):
    """bench.py's N>1 host logic under gloo: max-over-ranks timing and the row
    shards each rank draws (they tile N exactly)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    out = str(tmp_path / "bench")
    mp.spawn(_bench_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    t, n1, n2, N = np.load(out + ".npy")
    assert t == 1.5 + (world - 1)
    assert n1 == n2 == N
