"""Pins for the oracle's K-Means++ seeding (-m "not gpu", reading
R-A27 in DESIGN.md §2): SPEC.md:338-346's worked examples, closed-form inverse
CDF counts, scipy cdist for the fixed-point D^2, and the prefix property of the
sequential draw.
"""
import numpy as np
import pytest
from scipy.spatial.distance import cdist

import oracle


def test_k1_is_a_uniform_index():
    X = np.arange(7, dtype=np.float32)[:, None]
    for u0 in (0.0, 0.5, 0.99, 0.999999):
        assert list(oracle.seed_pp(X, 1, [u0])) == [int(np.floor(u0 * 7))]


def test_spec_worked_examples():
    # data {0, 0, 10}, first center 10 -> second is 0 with probability 1,
    # each duplicate equally likely (weights 100, 100, 0)
    X = np.array([[0], [0], [10]], np.float32)
    assert list(oracle.seed_pp(X, 2, [0.9, 0.0])) == [2, 0]
    assert list(oracle.seed_pp(X, 2, [0.9, 0.4999])) == [2, 0]
    assert list(oracle.seed_pp(X, 2, [0.9, 0.5])) == [2, 1]
    assert list(oracle.seed_pp(X, 2, [0.9, 0.9999])) == [2, 1]
    # {0, 1, 3} from center 0: D^2 = (0, 1, 9) -> P = (0, 0.1, 0.9); u in [0, 0.1) -> 1
    X = np.array([[0], [1], [3]], np.float32)
    assert list(oracle.seed_pp(X, 2, [0.0, 0.0999])) == [0, 1]
    assert list(oracle.seed_pp(X, 2, [0.0, 0.1])) == [0, 2]
    assert list(oracle.seed_pp(X, 3, [0.0, 0.5, 0.7])) == [0, 2, 1]


def test_inverse_cdf_counts_are_proportional_to_d2():
    # 1-D {0, 1, 2, 4}, center 0: D^2 = (0, 1, 4, 16) exactly; a midpoint grid of
    # 2100 uniforms lands 100 / 400 / 1600 times on samples 1 / 2 / 3
    X = np.array([[0], [1], [2], [4]], np.float32)
    counts = np.zeros(4, int)
    for g in range(2100):
        counts[oracle.seed_pp(X, 2, [0.0, (g + 0.5) / 2100])[1]] += 1
    assert list(counts) == [0, 100, 400, 1600]


def test_duplicates_and_too_few_distinct_points():
    # one value duplicated, k = 2 over 2 distinct values -> the second
    # center is always the other value; k above the number of distinct values is an error
    X = np.array([[1.5]] * 5 + [[-2.0]] * 3, np.float32)
    rng = np.random.default_rng(0)
    for _ in range(50):
        u = rng.random(2)
        i0, i1 = oracle.seed_pp(X, 2, u)
        assert X[i0, 0] != X[i1, 0]
    with pytest.raises(oracle.SeedError):
        oracle.seed_pp(X, 3, [0.1, 0.2, 0.3])
    with pytest.raises(oracle.SeedError):
        oracle.seed_pp(X, 2, [0.1, 1.0])
    with pytest.raises(oracle.SeedError):
        oracle.seed_pp(X, 9, np.zeros(9))


@pytest.mark.parametrize("N,d,k", [(300, 7, 10), (2000, 128, 6), (500, 1, 25)])
def test_fixed_point_d2_matches_cdist(N, d, k):
    """The final D2 equals min_j ||x - x_idx_j||^2 2^t to within d/2 units (one
    rounding per term); chosen samples are distinct with D2 = 0; (2000, 128)
    exercises the weight shift (bitlen(M) + ceil(log2 N) > 62)."""
    rng = np.random.default_rng(N + d)
    X = (rng.normal(0, 3, (N, d)) + rng.integers(-5, 5, (N, 1))).astype(np.float32)
    u = rng.random(k)
    idx, D2 = oracle.seed_pp(X, k, u, return_d2=True)
    assert len(set(idx.tolist())) == k
    t = oracle.seed_scale(X)
    ref = cdist(X.astype(np.float64), X[idx].astype(np.float64), "sqeuclidean").min(axis=1) * 2.0 ** t
    assert np.all(np.abs(D2 - ref) <= d / 2 + 1e-9 * ref)
    assert np.all(D2[idx] == 0)


@pytest.mark.parametrize("N,d", [(400, 3), (2000, 128)])
def test_sequential_prefix_and_positive_weight(N, d):
    """Drawing k centers repeats the (k-1)-center draw as its prefix, and every new
    center had D2 > 0 when it was drawn (D^2 = 0 samples are never chosen)."""
    rng = np.random.default_rng(7 * N + d)
    X = rng.normal(0, 1, (N, d)).astype(np.float32)
    X[N // 2:] = X[: N - N // 2]                     # every sample duplicated
    u = rng.random(12)
    full = oracle.seed_pp(X, 12, u)
    for r in range(1, 12):
        idx, D2 = oracle.seed_pp(X, r, u[:r], return_d2=True)
        assert list(idx) == list(full[:r])
        assert D2[full[r]] > 0


def test_shifted_weights_follow_d2():
    """Under the weight shift the draw frequencies still follow D^2 / sum D^2
    (scipy distances) to the grid resolution."""
    rng = np.random.default_rng(3)
    N, d = 80, 128
    X = rng.normal(0, 1, (N, d)).astype(np.float32)
    X[:40] *= 3.0
    G = 4000
    counts = np.zeros(N)
    for g in range(G):
        counts[oracle.seed_pp(X, 2, [0.0, (g + 0.5) / G])[1]] += 1
    p = cdist(X.astype(np.float64), X[:1].astype(np.float64), "sqeuclidean")[:, 0]
    p /= p.sum()
    assert np.abs(counts / G - p).max() <= 1.5 / G
