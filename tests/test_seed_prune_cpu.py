"""-m "not gpu": the skip rule of the pruned K-Means++ D^2 update (seed.cu
k_seed_dist_pr) restated here and checked against the
definition of the fixed-point distance (reading R-A27):

    dist_i(c) = sum_k rint(fl(fl(x_ik - c_k)^2) 2^t)          (int64)

A row is skipped for the newest center c_q when, with j = near_i and
D2_i = dist_i(c_j),

    cc_lo(q, j) >= 2 a_up (1 + 1e-9),
    a_up = sqrt((D2_i + d) 2^-t (1 + 1e-12)) (1 + 1e-12),
    cc_lo = sqrt(sum_k (c_qk - c_jk)^2) (1 - 1e-9).

The kernel's claim: every skipped row has dist_i(c_q) >= D2_i, so the minimum
(and the draw) is unchanged.  Checked on random clustered data (where the rule
fires often) and on rows placed at the triangle-inequality boundary (x at the
midpoint of c_j and c_q, nudged both ways), where a missing margin would show.
"""
import numpy as np
import pytest

import oracle


def fx_dist(X, c, t):
    df = X.astype(np.float64) - c.astype(np.float64)[None, :]
    return np.rint((df * df) * 2.0 ** t).astype(np.int64).sum(1)


def skip_rule(D2, cq, cj, d, t):
    a_up = np.sqrt((D2.astype(np.float64) + d) * 2.0 ** (-t) * (1.0 + 1e-12)) * (1.0 + 1e-12)
    cc = np.sqrt(((cq.astype(np.float64) - cj.astype(np.float64)) ** 2).sum()) * (1.0 - 1e-9)
    return cc >= 2.0 * a_up * (1.0 + 1e-9)


def run_rounds(X, centers, t):
    """D2 / near after the given centers, checking every skip on the way."""
    d = X.shape[1]
    D2 = fx_dist(X, X[centers[0]], t)
    near = np.zeros(len(X), np.int64)
    skipped = 0
    for q in range(1, len(centers)):
        cq = X[centers[q]]
        dq = fx_dist(X, cq, t)
        for j in np.unique(near):
            rows = np.nonzero(near == j)[0]
            sk = rows[skip_rule(D2[rows], cq, X[centers[j]], d, t)]
            assert (dq[sk] >= D2[sk]).all(), (q, j)          # the minimum cannot change
            skipped += len(sk)
        upd = dq < D2
        D2 = np.where(upd, dq, D2)
        near = np.where(upd, q, near)
    return D2, skipped


@pytest.mark.parametrize("seed,d", [(0, 4), (1, 16), (2, 64)])
def test_skip_rule_never_changes_a_minimum(seed, d):
    rng = np.random.default_rng(seed)
    mu = rng.uniform(-50, 50, (12, d))
    X = (mu[rng.integers(0, 12, 6000)] + rng.normal(0, 1.0, (6000, d))).astype(np.float32)
    t = oracle.seed_scale(X)
    centers = rng.choice(len(X), 24, replace=False)
    D2, skipped = run_rounds(X, centers, t)
    assert skipped > len(X)                                   # the rule does fire on clustered data
    # the pruned sequence ends at the exact minimum over all centers
    full = np.min(np.stack([fx_dist(X, X[c], t) for c in centers]), 0)
    assert (D2 == full).all()


@pytest.mark.parametrize("scale", [1e-3, 1.0, 1e3])
def test_skip_rule_at_the_boundary(scale):
    # c_j = 0, c_q = v, x = v / 2 (1 +- eps): ||c_q - c_j|| = 2 ||x - c_j|| up to eps,
    # the case the margins exist for
    rng = np.random.default_rng(7)
    d = 8
    v = (rng.normal(0, 1, d) * scale).astype(np.float32)
    cj = np.zeros(d, np.float32)
    rows = []
    for eps in (-1e-3, -1e-6, -1e-9, 0.0, 1e-9, 1e-6, 1e-3):
        rows.append((v.astype(np.float64) / 2 * (1 + eps)).astype(np.float32))
    X = np.stack(rows + [v, cj]).astype(np.float32)
    t = oracle.seed_scale(X)
    D2 = fx_dist(X, cj, t)
    dq = fx_dist(X, v, t)
    sk = skip_rule(D2, v, cj, d, t)
    assert (dq[sk] >= D2[sk]).all()
    # rows at or past the midpoint (within the 1e-9 margin) are never skipped; a row
    # clearly on c_j's side is (the rule is not vacuous)
    assert not sk[2:7].any()
    assert sk[0]
