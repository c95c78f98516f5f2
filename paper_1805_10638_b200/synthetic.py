"""Seeded synthetic inputs for the five BASELINE.json configs (c1..c5).

This module holds NO arithmetic of the method: it only draws samples X and
the initial centroids C^0 (K distinct samples, BASELINE.json "init = K random
samples").  It is the one module shared by the oracle tests and the CUDA-path
tests/bench (task rule ③); it imports neither side.

The paper's datasets (Table 1) are not in this container;
these seeded generators stand in for them (DESIGN.md §4 gives the recipe and
which paper dataset each config plays the role of).

Determinism: every random stream is a numpy ``default_rng`` seeded from
``SeedSequence([180510638, cfg, seed, stream, ...])``; large configs are drawn
in fixed 2^20-row chunks, each with its own stream, so the bytes do not
depend on thread count.
"""
from __future__ import annotations

import concurrent.futures as cf
import dataclasses
import os

import threading

import numpy as np

TAG = 180510638
CHUNK = 1 << 20


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    N: int
    d: int
    K: int
    m0: int = 5           # BASELINE.json configs[0] says m0 = 5; reading R-A18 applies it to all
    well_separated: bool = True


CONFIGS = {
    "c1": Config("c1", 10_000, 2, 10),
    "c2": Config("c2", 100_000, 16, 64),
    "c3": Config("c3", 1_000_000, 32, 256, well_separated=False),
    "c4": Config("c4", 4_000_000, 128, 1024),
    "c5": Config("c5", 16_000_000, 64, 4096, well_separated=False),
}
CFG_INDEX = {"c1": 1, "c2": 2, "c3": 3, "c4": 4, "c5": 5}


# numpy's BLAS (OpenBLAS) corrupted c4 rows when the chunk threads multiplied
# concurrently (different bytes run to run); the matmuls are serialised.
_BLAS_LOCK = threading.Lock()


def _rng(cfg: str, seed: int, *stream):
    return np.random.default_rng(np.random.SeedSequence([TAG, CFG_INDEX[cfg], seed, *stream]))


def zipf_sizes(N: int, K: int, s: float = 1.1) -> np.ndarray:
    """n_k proportional to k^-s over ranks k = 1..K, rounded by largest remainder to sum to N."""
    w = np.arange(1, K + 1, dtype=np.float64) ** (-s)
    q = w / w.sum() * N
    n = np.floor(q).astype(np.int64)
    rem = N - int(n.sum())
    order = np.argsort(-(q - n), kind="stable")
    n[order[:rem]] += 1
    return n


def _params(cfg: str, seed: int, N: int, d: int, K: int):
    """Per-config mixture parameters and the per-row component vector (params stream 0)."""
    r = _rng(cfg, seed, 0)
    p: dict = {}
    if cfg == "c1":
        p["mu"] = r.uniform(-10, 10, size=(K, d))
        p["z"] = r.integers(0, K, size=N)
    elif cfg == "c2":
        p["mu"] = r.uniform(-20, 20, size=(K, d))
        p["sig"] = r.uniform(0.5, 3.0, size=(K, d))
        w = r.dirichlet(np.ones(K))
        p["z"] = r.choice(K, size=N, p=w)
    elif cfg == "c3":
        n_mix = int(round(0.7 * N))
        p["mu"] = 5.0 * r.standard_normal((K, d))           # N(0, 25 I)
        p["sig"] = r.uniform(0.5, 2.0, size=K)
        kind = np.zeros(N, dtype=np.int8); kind[n_mix:] = 1    # 1 = background noise
        p["kind"] = r.permutation(kind)
        p["z"] = r.integers(0, K, size=N)                    # equal weights
    elif cfg == "c4":
        Q, _ = np.linalg.qr(r.standard_normal((d, 16)))
        p["Q"] = Q
        p["mu"] = r.uniform(-20, 20, size=(K, 16)) @ Q.T     # means on a 16-dim subspace
        sizes = zipf_sizes(N, K, 1.1)
        comp = r.permutation(K)                              # rank -> component
        p["z"] = r.permutation(np.repeat(comp, sizes))
    elif cfg == "c5":
        pass
    else:
        raise KeyError(cfg)
    return p


def _chunk(cfg: str, seed: int, c: int, r0: int, r1: int, d: int, p: dict) -> np.ndarray:
    r = _rng(cfg, seed, 2, c)
    n = r1 - r0
    if cfg == "c1":
        x = p["mu"][p["z"][r0:r1]] + r.standard_normal((n, d))
    elif cfg == "c2":
        z = p["z"][r0:r1]
        x = p["mu"][z] + p["sig"][z] * r.standard_normal((n, d))
    elif cfg == "c3":
        z = p["z"][r0:r1]
        g = p["mu"][z] + p["sig"][z][:, None] * r.standard_normal((n, d))
        u = r.uniform(-15.0, 15.0, size=(n, d))
        x = np.where((p["kind"][r0:r1] == 1)[:, None], u, g)
    elif cfg == "c4":
        Q = p["Q"]
        z = p["z"][r0:r1]
        a = r.standard_normal((n, 16))
        b = r.standard_normal((n, d))
        with _BLAS_LOCK:                                      # BLAS is not safe under concurrent callers here
            off = b - (b @ Q) @ Q.T                           # (I - Q Q^T) b
            aq = a @ Q.T
        x = p["mu"][z] + aq + 0.1 * off
    elif cfg == "c5":
        return r.random((n, d), dtype=np.float32)
    return x.astype(np.float32)


def make(cfg: str, seed: int = 0, N: int | None = None, K: int | None = None,
         threads: int | None = None):
    """Return (X float32 [N, d], C0 float32 [K, d], Config).

    N / K override the config's sizes with the same distribution (smaller
    parity cases)."""
    base = CONFIGS[cfg]
    N = base.N if N is None else int(N)
    K = base.K if K is None else int(K)
    d = base.d
    if K > N:
        raise ValueError("K > N")
    p = _params(cfg, seed, N, d, K)
    X = np.empty((N, d), dtype=np.float32)
    bounds = [(c, r0, min(r0 + CHUNK, N)) for c, r0 in enumerate(range(0, N, CHUNK))]
    nthreads = threads or min(len(bounds), os.cpu_count() or 1, 16)

    def work(b):
        c, r0, r1 = b
        X[r0:r1] = _chunk(cfg, seed, c, r0, r1, d, p)

    if nthreads > 1 and len(bounds) > 1:
        with cf.ThreadPoolExecutor(nthreads) as ex:
            list(ex.map(work, bounds))
    else:
        for b in bounds:
            work(b)
    idx = _rng(cfg, seed, 1).choice(N, K, replace=False)
    C0 = X[idx].copy()
    return X, C0, dataclasses.replace(base, N=N, K=K)


def make_shard(cfg: str, rank: int, world: int, seed: int = 0, N: int | None = None, K: int | None = None):
    """(X[lo:hi] of shard_bounds(N, rank, world), C0, Config): the same bytes as
    make(...) restricted to this rank's rows, without holding the full X (each
    chunk is drawn, its shard rows and C^0 rows are kept, the rest dropped)."""
    base = CONFIGS[cfg]
    N = base.N if N is None else int(N)
    K = base.K if K is None else int(K)
    d = base.d
    if K > N:
        raise ValueError("K > N")
    lo, hi = shard_bounds(N, rank, world)
    p = _params(cfg, seed, N, d, K)
    idx = _rng(cfg, seed, 1).choice(N, K, replace=False)
    Xs = np.empty((hi - lo, d), dtype=np.float32)
    C0 = np.empty((K, d), dtype=np.float32)
    bounds = [(c, r0, min(r0 + CHUNK, N)) for c, r0 in enumerate(range(0, N, CHUNK))]
    need = [b for b in bounds if (b[1] < hi and b[2] > lo) or np.any((idx >= b[1]) & (idx < b[2]))]
    nthreads = max(1, min(len(need), (os.cpu_count() or 1) // max(world, 1), 16))

    def work(b):
        c, r0, r1 = b
        x = _chunk(cfg, seed, c, r0, r1, d, p)
        a0, a1 = max(r0, lo), min(r1, hi)
        if a0 < a1:
            Xs[a0 - lo:a1 - lo] = x[a0 - r0:a1 - r0]
        sel = np.nonzero((idx >= r0) & (idx < r1))[0]
        C0[sel] = x[idx[sel] - r0]

    if nthreads > 1 and len(need) > 1:
        with cf.ThreadPoolExecutor(nthreads) as ex:
            list(ex.map(work, need))
    else:
        for b in need:
            work(b)
    return Xs, C0, dataclasses.replace(base, N=N, K=K)


def shard_bounds(N: int, rank: int, world: int):
    """Contiguous row block of `rank` (data-parallel sharding over samples)."""
    q, r = divmod(N, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def seed_uniforms(cfg: str, K: int, seed: int = 0) -> np.ndarray:
    """K uniforms in [0, 1) for K-Means++ seeding (kmeans_seed_pp / oracle.seed_pp),
    from their own stream (3) of the config's seed sequence."""
    return _rng(cfg, seed, 3).random(K)

