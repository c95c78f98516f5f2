"""-m gpu: K-Means++ seeding on the device (kmeans_seed_pp) against
the oracle's ora_seed_pp with the same uniforms: the drawn indices are
bit-exact (integer D^2 weights, reading R-A27) and C0 holds exactly those rows.
Covers every dist kernel (d = 4 LPR for LPR = 1..32, and any other d) and the
"fewer distinct samples than K" error."""
import numpy as np
import pytest

import oracle
from gpu_helpers import dev, make, require_gpu, torch
from paper_1805_10638_b200 import aakm, synthetic

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu():
    require_gpu()


def seed_both(X, K, u):
    km = aakm.KMeans(dev(X), K, aakm.config())
    C, idx = km.seed_pp(u)
    km.close()
    ref = oracle.seed_pp(X, K, u)
    return C.cpu().numpy(), idx, ref


@pytest.mark.parametrize("cfg,N,K", [("c1", None, None), ("c2", None, None), ("c3", 30_011, 64),
                                     ("c4", 8_003, 64), ("c5", 20_000, 256)])
def test_seed_parity_configs(cfg, N, K):
    X, _, c = make(cfg, N=N, K=K)
    u = synthetic.seed_uniforms(cfg, c.K)
    C, idx, ref = seed_both(X, c.K, u)
    np.testing.assert_array_equal(idx, ref)
    np.testing.assert_array_equal(C, X[ref])


@pytest.mark.parametrize("d", [4, 8, 7, 1, 33, 128])
def test_seed_parity_dims(d):
    rng = np.random.default_rng(40 + d)
    n, K = 5_000, 40
    X = (rng.normal(0, 2, (n, d)) + rng.integers(-4, 4, (n, 1)) * 5).astype(np.float32)
    X[100:200] = X[0]                                  # duplicates of the first rows
    u = rng.random(K)
    C, idx, ref = seed_both(X, K, u)
    np.testing.assert_array_equal(idx, ref)
    np.testing.assert_array_equal(C, X[ref])


def test_seed_full_size_prefix():
    """BASELINE full sizes: the first centers of c4 (4 M x 128) and c5 (16 M x 64)."""
    for cfg, K in (("c4", 4), ("c5", 3)):
        X, _, c = make(cfg)
        u = synthetic.seed_uniforms(cfg, K)
        km = aakm.KMeans(dev(X), K, aakm.config())
        C, idx = km.seed_pp(u)
        km.close()
        ref = oracle.seed_pp(X, K, u)
        np.testing.assert_array_equal(idx, ref)
        np.testing.assert_array_equal(C.cpu().numpy(), X[ref])
        del X
        torch.cuda.empty_cache()


def test_seed_errors_and_repeatability():
    X = np.array([[1.5, 0.0]] * 50 + [[-2.0, 1.0]] * 30, np.float32)
    km = aakm.KMeans(dev(X), 3, aakm.config())
    with pytest.raises(aakm.AAKMError):
        km.seed_pp([0.1, 0.5, 0.7])                    # only 2 distinct samples
    with pytest.raises(aakm.AAKMError):
        km.seed_pp([0.1, 0.5, 1.0])                    # u outside [0, 1)
    km.close()
    km = aakm.KMeans(dev(X), 2, aakm.config())
    C1, i1 = km.seed_pp([0.3, 0.6])
    C2, i2 = km.seed_pp([0.3, 0.6])
    assert list(i1) == list(i2) == list(oracle.seed_pp(X, 2, [0.3, 0.6]))
    assert X[i1[0], 0] != X[i1[1], 0]
    km.close()


def test_seeded_run_matches_oracle():
    """Seeding feeds Algorithm 1: C0 from kmeans_seed_pp, then kmeans_run, vs
    the oracle's seed + run (same iteration count and energy)."""
    X, _, c = make("c2", N=20_000, K=32)
    u = synthetic.seed_uniforms("c2", 32)
    km = aakm.KMeans(dev(X), 32, aakm.config(m0=5))
    C0, idx = km.seed_pp(u)
    C, labs, rep = km.run(C0)
    km.close()
    ref_idx = oracle.seed_pp(X, 32, u)
    np.testing.assert_array_equal(idx, ref_idx)
    ref = oracle.run(X, X[ref_idx].astype(np.float64), oracle.OracleConfig(m0=5))
    assert rep["converged"] and ref["converged"]
    assert rep["iters"] == ref["iters"]
    assert abs(rep["energy"] - ref["energy"]) <= 1e-6 * ref["energy"]


def test_seed_k1_and_k_equals_n():
    """K = 1 is one uniform index; K = N over distinct rows draws every row once
    (each round picks a remaining row with D^2 > 0), in the oracle's order."""
    rng = np.random.default_rng(5)
    X = rng.normal(0, 1, (300, 8)).astype(np.float32)
    for K in (1, 300):
        u = rng.random(K)
        C, idx, ref = seed_both(X, K, u)
        np.testing.assert_array_equal(idx, ref)
        np.testing.assert_array_equal(C, X[ref])
        if K == 300:
            assert sorted(idx.tolist()) == list(range(300))
