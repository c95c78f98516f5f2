"""Pins for the CPU oracle (-m "not gpu").  Each test ties an oracle function
to something other than itself: a worked example, a closed form, a library
routine, brute force, or an invariant the paper proves.  See DESIGN.md §3.
"""
import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def fr(v):
    return float(Fraction(v))


# ---------------------------------------------------------------- O1 assign
def test_assign_worked_examples():
    # SPEC.md:99-101 ([DERIVED]/[TRIVIAL]); Eq. 3
    assert list(oracle.assign([0, 1, 4, 5], [0, 5])) == [0, 0, 1, 1]
    assert list(oracle.assign([0, 1, 4, 5], [3.0])) == [0, 0, 0, 0]          # K = 1
    assert list(oracle.assign([2.0], [1, 3])) == [0]                         # exact tie -> lowest index (R-A16)
    assert list(oracle.assign([2.0], [3, 1])) == [0]


@pytest.mark.parametrize("d,K", [(1, 3), (2, 10), (16, 64), (33, 7)])
def test_assign_matches_cdist_argmin(d, K):
    from scipy.spatial.distance import cdist
    rng = np.random.default_rng(d * 100 + K)
    X = rng.standard_normal((2000, d)).astype(np.float32)
    C = rng.standard_normal((K, d))
    D = cdist(X.astype(np.float64), C, "sqeuclidean")
    ref = D.argmin(1)
    got = oracle.assign(X, C)
    srt = np.sort(D, axis=1)
    clear = (srt[:, 1] - srt[:, 0]) > 1e-9 * (1 + srt[:, 0]) if K > 1 else np.ones(len(X), bool)
    assert clear.mean() > 0.99
    np.testing.assert_array_equal(got[clear], ref[clear])
    b1, b2 = oracle.best2(X, C)
    np.testing.assert_allclose(b1, srt[:, 0], rtol=1e-12, atol=1e-12)
    if K > 1:
        np.testing.assert_allclose(b2, srt[:, 1], rtol=1e-12, atol=1e-12)


def test_sqdist_direct_difference():
    # direct differences are exact on small integers (Eq. 1 term)
    assert oracle.sqdist([1, 2, 3], [4, 6, 3]) == 25.0


def _all_labelings(N, K):
    return itertools.product(range(K), repeat=N)


@settings(max_examples=25, deadline=None)
@given(st.integers(0, 10**6))
def test_assign_minimizes_energy_over_all_labelings(seed):
    # SPEC.md:61 invariant; the nearest assignment is the minimizer of Eq. 2 over rho for fixed C
    rng = np.random.default_rng(seed)
    N, K, d = 6, 3, 2
    X = rng.integers(-5, 6, size=(N, d)).astype(np.float32)
    C = rng.integers(-5, 6, size=(K, d)).astype(np.float64)
    lab = oracle.assign(X, C)
    e_near = oracle.energy(X, C, lab)
    e_min = min(oracle.energy(X, C, np.array(p, np.int32)) for p in _all_labelings(N, K))
    assert e_near == e_min


def test_assign_permutation_invariance():
    # permuting samples permutes labels
    rng = np.random.default_rng(3)
    X = rng.standard_normal((500, 4)).astype(np.float32)
    C = rng.standard_normal((9, 4))
    perm = rng.permutation(500)
    np.testing.assert_array_equal(oracle.assign(X[perm], C), oracle.assign(X, C)[perm])


# ---------------------------------------------------------------- O2 energy
def test_energy_worked_examples():
    # SPEC.md:56-58
    assert oracle.energy([0, 1, 4, 5], [0.5, 4.5], [0, 0, 1, 1]) == 1.0
    # SPEC.md:58 prints "4+2.25+2.25+6.25 = 14.75"; its first term is a slip:
    # (0-2.5)^2 = 6.25, so the given-assignment total is 6.25+2.25+2.25+6.25 = 17 (DESIGN.md R-S1)
    assert oracle.energy([0, 1, 4, 5], [2.5, 99], [0, 0, 0, 0]) == 17.0
    X = np.array([[0, 1], [2, 3], [4, 5]], np.float32)
    assert oracle.energy(X, X.astype(np.float64), [0, 1, 2]) == 0.0     # K = N, C = X


def test_energy_matches_library_sum():
    from scipy.spatial.distance import cdist
    rng = np.random.default_rng(5)
    X = rng.standard_normal((3000, 8)).astype(np.float32)
    C = rng.standard_normal((20, 8))
    lab = rng.integers(0, 20, 3000).astype(np.int32)
    ref = cdist(X.astype(np.float64), C, "sqeuclidean")[np.arange(3000), lab].sum()
    assert abs(oracle.energy(X, C, lab) - ref) <= 1e-12 * ref


def test_surrogate_majorizes_energy():
    # Eq. 5: E(C) <= Ebar^t(C) for all C, equality at C^t
    rng = np.random.default_rng(11)
    X = rng.standard_normal((800, 3)).astype(np.float32)
    Ct = rng.standard_normal((6, 3))
    Pt = oracle.assign(X, Ct)
    for _ in range(20):
        C = Ct + rng.standard_normal(Ct.shape)
        E = oracle.energy(X, C, oracle.assign(X, C))
        Ebar = oracle.energy(X, C, Pt)
        assert E <= Ebar
    assert oracle.energy(X, Ct, oracle.assign(X, Ct)) == oracle.energy(X, Ct, Pt)


# ---------------------------------------------------------------- O3 update
def test_update_worked_examples():
    # SPEC.md:172-174, Eq. 4, empty-cluster reading R-A15
    G, n = oracle.update([0, 1, 4, 5], [0, 0, 1, 1], [0.0, 5.0])
    assert G.ravel().tolist() == [0.5, 4.5] and n.tolist() == [2, 2]
    G, n = oracle.update([0, 1, 4, 5], [0, 0, 0, 0], [2.5, 99.0])
    assert G.ravel().tolist() == [2.5, 99.0] and n.tolist() == [4, 0]
    X = np.array([[1, 2], [3, 4], [5, 6]], np.float32)
    G, _ = oracle.update(X, [0, 1, 2], np.zeros((3, 2)))
    np.testing.assert_array_equal(G, X)


def test_update_matches_bincount_means():
    rng = np.random.default_rng(7)
    X = rng.standard_normal((5000, 5)).astype(np.float32)
    lab = rng.integers(0, 30, 5000).astype(np.int32)
    lab[lab == 13] = 12                                   # cluster 13 empty
    Cp = rng.standard_normal((30, 5))
    G, n = oracle.update(X, lab, Cp)
    cnt = np.bincount(lab, minlength=30)
    S = np.zeros((30, 5)); np.add.at(S, lab, X.astype(np.float64))
    ref = np.where(cnt[:, None] > 0, S / np.maximum(cnt, 1)[:, None], Cp)
    np.testing.assert_array_equal(n, cnt)
    np.testing.assert_allclose(G, ref, rtol=1e-13, atol=1e-14)


def test_G_fixed_point_and_global_mean():
    # {0.5,4.5} is a fixed point of G; K=1 -> global mean
    X = [0, 1, 4, 5]
    G, _ = oracle.update(X, oracle.assign(X, [0.5, 4.5]), [0.5, 4.5])
    assert G.ravel().tolist() == [0.5, 4.5]
    G, _ = oracle.update(X, oracle.assign(X, [17.0]), [17.0])
    assert G.ravel().tolist() == [2.5]


# ---------------------------------------------------------------- O11 least squares
def test_ls_closed_forms():
    # SPEC.md:246-248; Eq. 7
    th, used = oracle.ls_solve([[1.0, 2.0, -1.0]], [1.0, 2.0, -1.0])
    assert used == 1 and abs(th[0] - 1.0) < 1e-9
    th, _ = oracle.ls_solve([[1.0, 1.0]], [1.0, 0.0])
    assert abs(th[0] - 0.5) < 1e-9
    th, _ = oracle.ls_solve([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]], [1.0, 1.0, 0.0])
    np.testing.assert_allclose(th, [1.0, 1.0], atol=1e-9)
    # m = 1 closed form: theta = <dF, F> / ||dF||^2
    rng = np.random.default_rng(2)
    dF, F = rng.standard_normal(50), rng.standard_normal(50)
    th, _ = oracle.ls_solve(dF[None], F)
    assert abs(th[0] - dF @ F / (dF @ dF)) < 1e-9 * abs(dF @ F / (dF @ dF))


@pytest.mark.parametrize("m_t,n", [(1, 10), (3, 64), (5, 64), (5, 40)])
def test_ls_matches_lstsq(m_t, n):
    # agree with numpy.linalg.lstsq on well-conditioned problems
    rng = np.random.default_rng(m_t * 1000 + n)
    dF = rng.standard_normal((m_t, n)); F = rng.standard_normal(n)
    ref = np.linalg.lstsq(dF.T, F, rcond=None)[0]
    th, used = oracle.ls_solve(dF, F)
    assert used == m_t
    np.testing.assert_allclose(th, ref, rtol=1e-8, atol=1e-10)


def test_ls_degenerate_columns():
    # R-A14: zero columns dropped; duplicate columns -> finite, residual-optimal theta
    th, used = oracle.ls_solve([[0.0, 0.0], [1.0, 1.0]], [1.0, 0.0])
    assert used == 1 and th[0] == 0.0 and abs(th[1] - 0.5) < 1e-9
    th, _ = oracle.ls_solve([[0.0, 0.0]], [1.0, 0.0])
    assert th.tolist() == [0.0]
    dF = np.array([[1.0, 2.0, 3.0], [1.0, 2.0, 3.0], [0.0, 1.0, 0.0]])
    F = np.array([2.0, 5.0, 6.0])
    th, _ = oracle.ls_solve(dF, F)
    assert np.all(np.isfinite(th))
    ref = np.linalg.lstsq(dF.T, F, rcond=None)[0]
    assert np.linalg.norm(F - dF.T @ th) <= np.linalg.norm(F - dF.T @ ref) + 1e-6
    # K*d < m (c1 has K*d = 20 < 30): more columns than dimensions
    rng = np.random.default_rng(9)
    dF = rng.standard_normal((6, 4)); F = rng.standard_normal(4)
    th, _ = oracle.ls_solve(dF, F)
    assert np.linalg.norm(F - dF.T @ th) < 1e-4 * np.linalg.norm(F)


# ---------------------------------------------------------------- O7 dynamic m
def test_adjust_m_rules():
    # Algorithm 1, constants PAPER.md:177; R-A5/R-A6
    # r = (E1 - Et)/(E2 - E1)
    assert oracle.adjust_m(5, 30, 9.99, 10.0, 11.0) == 4          # r = 0.01 < eps1
    assert oracle.adjust_m(0, 30, 9.99, 10.0, 11.0) == 0          # floor at 0
    assert oracle.adjust_m(30, 30, 9.4, 10.0, 11.0) == 30         # r = 0.6 > eps2 but capped
    assert oracle.adjust_m(5, 30, 9.4, 10.0, 11.0) == 6
    assert oracle.adjust_m(5, 30, 9.7, 10.0, 11.0) == 5           # r = 0.3 unchanged
    assert oracle.adjust_m(5, 30, 10.5, 10.0, 11.0) == 4          # energy increase -> r < 0 -> m-1
    assert oracle.adjust_m(5, 30, 9.0, 10.0, float("inf")) == 5   # E^{t-2} = +inf (t = 2)
    assert oracle.adjust_m(5, 30, 9.0, float("inf"), float("inf")) == 5
    assert oracle.adjust_m(5, 30, 9.0, 10.0, 10.0) == 5           # D = 0
    assert oracle.adjust_m(5, 30, 9.0, 10.0, 9.0) == 5            # D < 0


# ---------------------------------------------------------------- Algorithm 1 end to end
def _load_gold():
    with open(os.path.join(GOLD, "appendix_a_trace.json")) as f:
        return json.load(f)


def test_appendix_a_trace_pass_by_pass():
    g = _load_gold()
    X = np.array(g["X"], np.float32)
    st_ = oracle.AAState(X, oracle.OracleConfig(m0=g["m0"]))
    st_.init(np.array(g["C0"], np.float64))
    assert st_.labels_prev.tolist() == g["init"]["P0"]
    np.testing.assert_allclose(st_.Ghist[0].ravel(), [fr(v) for v in g["init"]["G0"]], rtol=1e-14)
    np.testing.assert_allclose(st_.Fhist[0].ravel(), [fr(v) for v in g["init"]["F0"]], rtol=1e-14)
    for p in g["passes"]:
        np.testing.assert_allclose(st_.C.ravel(), [fr(v) for v in p["C"]], rtol=1e-8)
        rc = st_.step()
        info = st_.info()
        assert info["m"] == p["m"]
        assert info["rejected"] == p["rejected"]
        if p.get("converged"):
            assert rc == 1
            assert abs(info["E_cand"] - fr(p["E_candidate"])) < 1e-7 * fr(p["E_candidate"])
            assert st_.labels.tolist() == p["P"]
            assert info["E"] == fr(p["E"])
            break
        assert rc == 0
        assert st_.labels_prev.tolist() == p["P"]
        assert abs(info["E"] - fr(p["E"])) < 1e-8 * fr(p["E"])
        assert info["accepted"] == p["accepted"] and info["m_t"] == p["m_t"]
        np.testing.assert_allclose(info["theta"], [fr(v) for v in p["theta"]], rtol=1e-7)  # ridge 1e-10 (R-A14) perturbs theta
        np.testing.assert_allclose(st_.Ghist[0].ravel(), [fr(v) for v in p["G"]], rtol=1e-8)
        np.testing.assert_allclose(st_.Fhist[0].ravel(), [fr(v) for v in p["F"]], rtol=1e-7, atol=1e-9)
        np.testing.assert_allclose(st_.C.ravel(), [fr(v) for v in p["C_next"]], rtol=1e-8)


def test_appendix_a_result_and_lloyd():
    g = _load_gold()
    X = np.array(g["X"], np.float64)
    r = oracle.run(X, g["C0"], oracle.OracleConfig(m0=g["m0"]))
    res = g["result"]
    assert r["converged"] and r["C"].ravel().tolist() == [fr(v) for v in res["C"]]
    assert r["energy"] == fr(res["E"])
    for k in ("iters", "accepted", "rejected", "n_assign", "m_final"):
        assert r[k] == res[k], k
    lr = oracle.lloyd(X, g["C0"], trace=True)
    assert [t["E"] for t in lr["trace"]] == pytest.approx([fr(v) for v in g["lloyd"]["E"]], rel=1e-15)
    assert lr["iters"] == g["lloyd"]["iters"] and lr["n_assign"] == g["lloyd"]["n_assign"]
    assert lr["C"].ravel().tolist() == [fr(v) for v in g["lloyd"]["C"]]


def test_lloyd_spec_toy():
    # {0,1,4,5}, C0 = {0,5} -> {0.5,4.5}, E = 1, 2 iterations
    r = oracle.lloyd([0, 1, 4, 5], [0.0, 5.0])
    assert r["C"].ravel().tolist() == [0.5, 4.5] and r["energy"] == 1.0 and r["iters"] == 2


def test_lloyd_matches_sklearn():
    # library routine: sklearn Lloyd, tol=0 (strict convergence), same C0
    from sklearn.cluster import KMeans
    from paper_1805_10638_b200 import synthetic
    # sklearn relocates empty clusters, so use instances whose run keeps all K non-empty
    checked = 0
    for cfg, seed, N in (("c1", 0, 10000), ("c2", 2, 8000), ("c2", 3, 8000), ("c2", 4, 8000)):
        X, C0, _ = synthetic.make(cfg, seed=seed, N=N)
        r = oracle.lloyd(X, C0)
        if np.all(np.bincount(r["labels"], minlength=len(C0)) > 0):
            _check_sklearn(X, C0, r)
            checked += 1
    assert checked >= 2


def _check_sklearn(X, C0, r):
    from sklearn.cluster import KMeans
    km = KMeans(n_clusters=len(C0), init=C0.astype(np.float64), n_init=1, algorithm="lloyd",
                tol=0.0, max_iter=10000).fit(X.astype(np.float64))
    np.testing.assert_array_equal(km.labels_, r["labels"])
    np.testing.assert_allclose(km.cluster_centers_, r["C"], rtol=1e-10, atol=1e-10)
    assert km.n_iter_ == r["iters"]
    assert abs(km.inertia_ - r["energy"]) <= 1e-9 * r["energy"]


@settings(max_examples=20, deadline=None)
@given(st.integers(0, 10**6), st.integers(0, 3), st.booleans())
def test_algorithm1_invariants(seed, m0, dynamic):
    # north_star invariants: Lloyd E monotone; accepted AA iterates never raise E;
    # m in [0, m_max]; the converged C is a fixed point of G and the mean of its members.
    rng = np.random.default_rng(seed)
    N, K, d = 300, 6, 2
    X = (rng.standard_normal((N, d)) + rng.integers(-3, 4, size=(N, d)) * 3).astype(np.float32)
    C0 = X[rng.choice(N, K, replace=False)].astype(np.float64)
    r = oracle.run(X, C0, oracle.OracleConfig(m0=m0, dynamic_m=dynamic, m_max=4), trace=True)
    assert r["converged"]
    Es = [t["E"] for t in r["trace"]]
    assert all(b <= a for a, b in zip(Es, Es[1:]))                # post-guard energies non-increasing
    assert all(0 <= t["m"] <= 4 for t in r["trace"])
    for t in r["trace"]:
        if t["accepted"]:
            assert t["E_cand"] == t["E"]
    G, n = oracle.update(X, r["labels"], r["C"])
    np.testing.assert_array_equal(G, r["C"])                    # fixed point (bitwise: same sums)
    np.testing.assert_array_equal(oracle.assign(X, r["C"]), r["labels"])
    assert r["energy"] == oracle.energy(X, r["C"], r["labels"])
    assert r["n_assign"] == r["iters"] + r["rejected"]


@settings(max_examples=15, deadline=None)
@given(st.integers(0, 10**6))
def test_m0_is_lloyd(seed):
    # fixed m = 0 reduces Algorithm 1 to Lloyd's algorithm, bitwise (R-A9)
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((400, 3)).astype(np.float32)
    C0 = X[rng.choice(400, 7, replace=False)].astype(np.float64)
    a = oracle.run(X, C0, oracle.OracleConfig(m0=0, dynamic_m=False), trace=True)
    # independent Lloyd loop built from the O1/O3 primitives
    C = C0.copy(); P = oracle.assign(X, C); C, _ = oracle.update(X, P, C); iters = 1
    while True:
        Pn = oracle.assign(X, C)
        if np.array_equal(Pn, P):
            break
        P = Pn; C, _ = oracle.update(X, P, C); iters += 1
    iters += 1
    np.testing.assert_array_equal(a["C"], C)
    assert a["iters"] == iters and a["rejected"] == 0 and a["accepted"] == 0


@settings(max_examples=10, deadline=None)
@given(st.integers(0, 10**6))
def test_final_energy_not_below_bruteforce_optimum(seed):
    # NP-hard problem: the method reaches a local minimum >= the global one,
    # enumerated over all K^N labelings for N <= 8, K <= 3
    rng = np.random.default_rng(seed)
    N, K = 8, 3
    X = rng.integers(-6, 7, size=(N, 1)).astype(np.float32)
    if len(np.unique(X)) < K:
        return
    C0 = np.unique(X)[:K].astype(np.float64)[:, None]
    r = oracle.run(X, C0, oracle.OracleConfig(m0=2))
    best = np.inf
    for lab in _all_labelings(N, K):
        lab = np.array(lab, np.int32)
        if len(np.unique(lab)) < K:
            continue
        G, _ = oracle.update(X, lab, np.zeros((K, 1)))
        best = min(best, oracle.energy(X, G, lab))
    assert r["energy"] >= best - 1e-12
    assert r["converged"]
