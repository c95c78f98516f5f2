"""-m gpu: the tensor-core assignment engines at shapes the main parity cases do
not reach -- ragged K (partial 256-centroid pair tiles and 128-centroid halves
past K), n with a partial last row-tile pair, the single-SM (cta_group::1)
variant -- each against the CPU oracle under the north-star tie rule."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from gpu_helpers import check_assign, dev, make, require_gpu, torch
from paper_1805_10638_b200 import aakm

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(autouse=True)
def _gpu():
    require_gpu()


@pytest.mark.parametrize("path,cfg", [("tc", "c3"), ("tc", "c5"), ("tc16", "c5"), ("tc16", "c4")])
# K = 2048 / 2049: the 2xFP16 engine's last four-splitter-warp tiling (8 accumulator
# tiles per row tile) and the first two-splitter one (9)
@pytest.mark.parametrize("K", [1, 100, 129, 257, 300, 1000, 2048, 2049])
def test_ragged_k(path, cfg, K):
    X, C0, c = make(cfg, N=3001, K=K)
    km = aakm.KMeans(dev(X), c.K, aakm.config(assign_path=path))
    rng = np.random.default_rng(K)
    C = C0 + rng.normal(0, 0.01, C0.shape)             # fp64 centroids (the ABI's state type)
    lab, E, _ = km.assign(dev(C))
    lab = lab.cpu().numpy()
    assert lab.min() >= 0 and lab.max() < c.K
    check_assign(X, C, lab, msg=f"{path}/{cfg}/K={K}")
    E_ora = oracle.energy(X, C.astype(np.float64), lab)
    assert abs(E - E_ora) <= 1e-6 * E_ora
    km.close()


@pytest.mark.parametrize("n", [128, 129, 255, 256, 257, 383, 385])
def test_row_tile_pairs(n):
    # 2-CTA pairs take row tiles two at a time: odd tile counts leave the partner
    # of the last pair with an all-out-of-bounds tile
    X, C0, c = make("c5", N=max(n, 300), K=100)
    X = X[:n]
    km = aakm.KMeans(dev(X), c.K, aakm.config(assign_path="tc16"))
    lab, _, _ = km.assign(dev(C0))
    check_assign(X, C0, lab.cpu().numpy(), msg=f"n={n}")
    km.close()


def test_single_sm_variant_subprocess():
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r); sys.path.insert(0, %r)
import oracle
from gpu_helpers import check_assign, dev, make
from paper_1805_10638_b200 import aakm
for path, cfg in (("tc16", "c5"), ("tc", "c3")):
    X, C0, c = make(cfg, N=5003, K=300)
    km = aakm.KMeans(dev(X), c.K, aakm.config(assign_path=path))
    lab, E, _ = km.assign(dev(C0))
    check_assign(X, C0, lab.cpu().numpy(), msg=path)
    C, lab, rep = km.run(dev(C0))
    assert rep["converged"], rep
    km.close()
print("ok")
""" % (ROOT, os.path.join(ROOT, "tests"))
    env = dict(os.environ, AAKM_TC_CG="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]


# ---------------------------------------------------------------- bounded engine (f2)
@pytest.mark.parametrize("cfg,N,K", [("c5", 40_000, 256), ("c4", 30_000, 256)])
def test_bounded_matches_dense_passes(cfg, N, K):
    """Hamerly-bounded assignment (cfg.bounded) against the dense engine, pass by
    pass from the same C^0: identical decisions and labels; energies to 1e-9."""
    X, C0, c = make(cfg, N=N, K=K)
    Xd = dev(X)
    kd = aakm.KMeans(Xd, c.K, aakm.config(m0=5, assign_path="tc16"))
    kb = aakm.KMeans(Xd, c.K, aakm.config(m0=5, assign_path="tc16", bounded=True))
    kd.aa_step(dev(C0)); kb.aa_step(dev(C0))
    for p in range(60):
        a, b = kd.aa_step(), kb.aa_step()
        for k in ("t", "m", "m_t", "accepted", "rejected", "converged", "changed"):
            assert a[k] == b[k], (p, k, a, b)
        assert abs(a["energy"] - b["energy"]) <= 1e-9 * a["energy"], (p, a, b)
        _, la = kd.centroids(); _, lb = kb.centroids()
        assert torch.equal(la, lb), p
        if a["converged"]:
            break
    scored, total = kb.bounded_stats()
    assert 0 < scored < total, (scored, total)      # the bounds did prove rows unchanged
    s0, t0 = kd.bounded_stats()
    assert s0 == t0
    kd.close(); kb.close()


@pytest.mark.parametrize("cfg,N,K,seed", [("c4", 8_000, 256, 0), ("c5", 20_000, 256, 1)])
def test_bounded_end_to_end_vs_oracle(cfg, N, K, seed):
    X, C0, c = make(cfg, seed=seed, N=N, K=K)
    km = aakm.KMeans(dev(X), c.K, aakm.config(m0=5, assign_path="tc16", bounded=True))
    C, lab, rep = km.run(dev(C0))
    ref = oracle.run(X, C0.astype(np.float64), oracle.OracleConfig(m0=5))
    assert rep["converged"] and ref["converged"]
    assert rep["iters"] == ref["iters"], (rep, ref["iters"])
    assert abs(rep["energy"] - ref["energy"]) <= 1e-4 * ref["energy"]
    check_assign(X, C.cpu().numpy(), lab.cpu().numpy())
    km.close()


# ---------------------------------------------------------------- checkpoint / resume
@pytest.mark.parametrize("cfg,N,K,path", [("c5", 30_000, 256, "auto"), ("c2", None, None, "auto"),
                                          ("c3", 20_000, 64, "tc")])
def test_checkpoint_resume(cfg, N, K, path):
    """kmeans_state_export after pass t, kmeans_state_import into a fresh handle on
    the same data: the resumed passes repeat the uninterrupted ones."""
    X, C0, c = make(cfg, N=N, K=K)
    Xd = dev(X)
    a = aakm.KMeans(Xd, c.K, aakm.config(m0=5, assign_path=path))
    a.aa_step(dev(C0))
    for _ in range(8):
        if a.aa_step()["converged"]:
            pytest.skip("converged before the checkpoint")
    snap = a.state_export()
    ref = [a.aa_step() for _ in range(6)]
    b = aakm.KMeans(Xd, c.K, aakm.config(m0=5, assign_path=path))
    b.state_import(snap)
    got = [b.aa_step() for _ in range(6)]
    for p, (x, y) in enumerate(zip(ref, got)):
        for k in ("t", "m", "m_t", "accepted", "rejected", "converged", "changed"):
            assert x[k] == y[k], (p, k, x, y)
        assert abs(x["energy"] - y["energy"]) <= 1e-9 * x["energy"], (p, x, y)
        if x["converged"]:
            break
    sa, sb = a.state_export(), b.state_export()
    assert np.allclose(sa["C"], sb["C"], rtol=1e-6, atol=1e-6)
    a.close(); b.close()


def test_state_import_validation():
    X, C0, c = make("c1")
    km = aakm.KMeans(dev(X), c.K, aakm.config(m0=2))
    km.aa_step(dev(C0)); km.aa_step()
    snap = km.state_export()
    bad = dict(snap, m=31)
    with pytest.raises(aakm.AAKMError):
        km.state_import(bad)
    km.close()


# ---------------------------------------------------------------- reproducibility
@pytest.mark.parametrize("cfg,N,K,bounded", [("c4", 40_000, 256, False), ("c5", 60_000, 512, True),
                                             ("c3", 50_000, 64, False)])
def test_runs_are_bitwise_reproducible(cfg, N, K, bounded):
    """The update sums are exact integers (order-free), the energy and the
    Anderson step fixed-order: two runs from the same C^0 agree bit for bit."""
    X, C0, c = make(cfg, N=N, K=K)
    Xd = dev(X)
    out = []
    for _ in range(2):
        km = aakm.KMeans(Xd, c.K, aakm.config(m0=5, bounded=bounded, max_iters=400))
        C, lab, rep = km.run(dev(C0))
        out.append((C.cpu().numpy().copy(), lab.cpu().numpy().copy(), rep))
        km.close()
    (C1, l1, r1), (C2, l2, r2) = out
    assert np.array_equal(C1.view(np.uint64), C2.view(np.uint64))
    assert np.array_equal(l1, l2)
    for k in ("iters", "n_assign", "n_accepted", "n_rejected", "converged", "m_final"):
        assert r1[k] == r2[k], k
    assert r1["energy"] == r2["energy"]


# ---------------------------------------------------------------- odd dimensions
@pytest.mark.parametrize("d", [1, 3, 7, 24, 33, 100])
def test_odd_d_assign_update_and_run(d):
    """d outside the synthetic configs: SIMT / 3xTF32 engines, the generic
    (non-float4) segmented sums at n >= 65 536 rows, and a short run vs the oracle."""
    rng = np.random.default_rng(d)
    n, K = 70_000, 37
    means = rng.normal(0, 4, (K, d))
    X = (means[rng.integers(0, K, n)] + rng.normal(0, 1, (n, d))).astype(np.float32)
    C0 = X[rng.choice(n, K, replace=False)].copy()
    km = aakm.KMeans(dev(X), K, aakm.config(m0=5))
    lab, E, _ = km.assign(dev(C0))
    lab = lab.cpu().numpy()
    check_assign(X, C0, lab, msg=f"d={d}")
    E_ora = oracle.energy(X, C0.astype(np.float64), lab)
    assert abs(E - E_ora) <= 1e-6 * E_ora
    G, cnt = km.update(dev(lab), dev(C0))
    G_ora, cnt_ora = oracle.update(X, lab, C0.astype(np.float64))
    np.testing.assert_array_equal(cnt.cpu().numpy(), cnt_ora)
    scale = np.maximum(np.abs(G_ora), np.sqrt(np.mean(G_ora ** 2)))
    assert (np.abs(G.cpu().numpy() - G_ora) / scale).max() <= 1e-6
    km.close()
    Xs, C0s = X[:4000], C0[:8]
    km = aakm.KMeans(dev(Xs), 8, aakm.config(m0=5))
    C, labs, rep = km.run(dev(C0s))
    ref = oracle.run(Xs, C0s.astype(np.float64), oracle.OracleConfig(m0=5))
    assert rep["converged"] and ref["converged"]
    assert rep["iters"] == ref["iters"] and abs(rep["energy"] - ref["energy"]) <= 1e-4 * ref["energy"]
    km.close()


# ---------------------------------------------------------------- degenerate shapes
def test_empty_shard_and_k_equals_n():
    """A rank with no rows (N < ranks) contributes nothing; K = n puts every
    sample on its own centroid (E = 0, labels = identity for distinct rows)."""
    X, C0, c = make("c4", N=300, K=300)
    X = np.unique(X, axis=0)[:256]
    n = len(X)
    # empty shard: partials are all zero, labels_prev/labels of length 0
    km = aakm.KMeans(torch.zeros((0, X.shape[1]), dtype=torch.float32, device="cuda"), 8, aakm.config(), n_global=n)
    part = km.update_partials(torch.zeros(0, dtype=torch.int32, device="cuda"), dev(X[:8])).cpu().numpy()
    assert not part.any()
    km.close()
    # K = n with C = X: exact identity labels, zero energy, G = X
    km = aakm.KMeans(dev(X), n, aakm.config(assign_path="tc16"))
    lab, E, _ = km.assign(dev(X))
    assert np.array_equal(lab.cpu().numpy(), np.arange(n)) and E == 0.0
    G, cnt = km.update(lab, dev(X))
    assert np.array_equal(G.cpu().numpy(), X) and (cnt.cpu().numpy() == 1).all()
    C, labs, rep = km.run(dev(X))
    assert rep["converged"] and rep["energy"] == 0.0 and rep["iters"] == 2
    km.close()


@pytest.mark.parametrize("d", [4, 8, 16, 32, 64, 128])
def test_sorted_update_engine(d):
    """The label-sorted update (n >= 65 536: histogram, scans, scatter, TMA
    gather4 segmented sums) for every float4 width: one cluster holding 40 % of
    the rows (hundreds of 256-row chunks), tiny and empty clusters, rows equal to
    their centroid (exact zero energy parts); S/N, E and #changed against the
    oracle (E to 1e-12: direct differences on both sides)."""
    rng = np.random.default_rng(100 + d)
    n, K = 70_001, 50
    X = rng.normal(0, 3, (n, d)).astype(np.float32)
    C = rng.normal(0, 3, (K, d)).astype(np.float32)
    lab = rng.integers(1, K - 3, n).astype(np.int32)              # K-3..K-1 stay empty
    lab[rng.random(n) < 0.4] = 0
    lab[:500] = 7
    X[:500] = C[7]                                                 # e_i = 0 exactly
    prev = lab.copy()
    prev[rng.random(n) < 0.1] = 1
    km = aakm.KMeans(dev(X), K, aakm.config())
    part = km.update_partials(dev(lab), dev(C), labels_prev=dev(prev)).cpu().numpy()
    G_ora, cnt = oracle.update(X, lab, C.astype(np.float64))
    np.testing.assert_array_equal(part[K * d:K * d + K], cnt)
    S = part[:K * d].reshape(K, d)
    G = np.where(cnt[:, None] > 0, S / np.maximum(cnt, 1)[:, None], C)
    np.testing.assert_allclose(G, G_ora, rtol=1e-12, atol=1e-12)
    E_ora = oracle.energy(X, C.astype(np.float64), lab)
    assert abs(part[-2] - E_ora) <= 1e-12 * E_ora, (part[-2], E_ora)
    assert part[-1] == float((lab != prev).sum())
    # the same through kmeans_update + kmeans_assign's energy on C itself
    G2, cnt2 = km.update(dev(lab), dev(C))
    np.testing.assert_array_equal(cnt2.cpu().numpy(), cnt)
    np.testing.assert_allclose(G2.cpu().numpy(), G_ora, rtol=1e-12, atol=1e-12)
    km.close()


@pytest.mark.parametrize("cfg,N,K,chunks,bounded", [("c5", 70_000, 512, 8, False), ("c4", 33_000, 256, 3, False),
                                                    ("c3", 50_001, 64, 64, False), ("c2", None, None, 4, False),
                                                    ("c5", 70_000, 512, 5, True)])
def test_streamed_host_pass_matches_resident(cfg, N, K, chunks, bounded):
    """kmeans_aa_step_host (X streamed from pinned host memory in row chunks under
    the assignment) repeats the resident passes bit for bit, even when the device
    copy of X was scrambled in between (the assignment must read the new rows)."""
    X, C0, c = make(cfg, N=N, K=K)
    a = aakm.KMeans(dev(X), c.K, aakm.config(m0=5, bounded=bounded))
    a.aa_step(dev(C0))
    ref = [a.aa_step() for _ in range(5)]
    sa = a.state_export()
    a.close()
    Xd = dev(X)
    b = aakm.KMeans(Xd, c.K, aakm.config(m0=5, bounded=bounded, x_refresh=True))
    b.aa_step(dev(C0))
    Xh = torch.from_numpy(X).pin_memory()
    got = []
    for _ in range(5):
        Xd.copy_(torch.randn_like(Xd))               # stale device rows: the pass must wait for the copy
        torch.cuda.synchronize()
        got.append(b.aa_step_host(Xh, chunks=chunks))
    sb = b.state_export()
    b.close()
    for x, y in zip(ref, got):
        assert x == y, (x, y)
    assert np.array_equal(sa["C"], sb["C"])


def test_streamed_host_pass_contract():
    """kmeans_aa_step_host is opt-in (cfg.x_refresh) and rejects rows outside the
    create-time range of X (the scales of every engine were derived from it)."""
    X, C0, c = make("c5", N=70_000, K=256)
    a = aakm.KMeans(dev(X), c.K, aakm.config(m0=5))
    a.aa_step(dev(C0))
    with pytest.raises(aakm.AAKMError):
        a.aa_step_host(torch.from_numpy(X).pin_memory())
    a.close()
    b = aakm.KMeans(dev(X), c.K, aakm.config(m0=5, x_refresh=True))
    b.aa_step(dev(C0))
    Xh = torch.from_numpy(X).pin_memory()
    b.aa_step_host(Xh)                                # same rows: fine
    Xh2 = Xh.clone()
    Xh2[123, 5] = 4.0                                 # c5 is U[0,1]: outside max |x|
    with pytest.raises(aakm.AAKMError):
        b.aa_step_host(Xh2)
    b.close()


@pytest.mark.parametrize("path", ["tc16", "tc"])
def test_exact_two_and_four_way_ties(path):
    """Rows at the exact midpoint of two centroids (two-centroid fast path on the
    2xFP16 engine) and at the centre of four equidistant centroids (candidate
    pass): the labels equal the oracle's lowest-index argmin bit for bit."""
    rng = np.random.default_rng(11)
    d, K = 64, 96
    C = (2 * rng.integers(-8, 9, (K, d))).astype(np.float32)      # even integers: midpoints exact
    n2 = 3000
    a = rng.integers(0, K, n2)
    b = (a + 1 + rng.integers(0, K - 1, n2)) % K
    X2 = (C[a] + C[b]) / 2                                        # ||x - c_a|| == ||x - c_b|| exactly
    # four centroids at +-2 e_p, +-2 e_q around a far-away centre: every one at distance 2
    base = np.full(d, 40.0, np.float32)
    C4 = np.stack([base + 2 * np.eye(d, dtype=np.float32)[0], base - 2 * np.eye(d, dtype=np.float32)[0],
                   base + 2 * np.eye(d, dtype=np.float32)[1], base - 2 * np.eye(d, dtype=np.float32)[1]])
    C = np.concatenate([C, C4]).astype(np.float32)
    X = np.concatenate([X2, np.repeat(base[None], 200, 0)]).astype(np.float32)
    km = aakm.KMeans(dev(X), C.shape[0], aakm.config(assign_path=path))
    lab, E, _ = km.assign(dev(C))
    km.close()
    ref = oracle.assign(X, C.astype(np.float64))
    np.testing.assert_array_equal(lab.cpu().numpy(), ref)
    assert (ref[n2:] == K).all()                                  # lowest index of the four


def test_assign_and_update_timing_hooks():
    """cfg.timing records one assignment and one update interval per main
    G-evaluation (branch A); both read back positive and reset on read."""
    X, C0, c = make("c5", N=70_000, K=256)
    km = aakm.KMeans(dev(X), c.K, aakm.config(m0=5, timing=True))
    km.aa_step(dev(C0))
    km.assign_timing(); km.update_timing()
    for _ in range(4):
        km.aa_step(info=False)
    a_ms, a_n = km.assign_timing()
    u_ms, u_n = km.update_timing()
    assert a_n == 4 and u_n == 4 and a_ms > 0 and u_ms > 0
    assert km.assign_timing() == (0.0, 0) and km.update_timing() == (0.0, 0)
    km.close()


@pytest.mark.parametrize("offset,d", [(0.0, 64), (30.0, 128), (300.0, 32)])
def test_sorted_energy_expansion_bound(offset, d):
    """Sorted engine energy (DESIGN R-A30): E = sum ||x_i||^2 + sum_j (N_j ||c_j||^2
    - 2 c_j . S_j) from the exact sums, against the oracle's direct differences,
    within the stated bound: every x_ik^2 and every (j, k) piece rounds once to the
    energy grid (<= half a unit of 2^-30/q each), plus 1e-13 E for the oracle's own
    fp64 rounding.  offset > 0 puts the data far from the origin (||x||^2 >> e_i:
    the expansion's cancellation case)."""
    rng = np.random.default_rng(7 + d)
    n, K = 70_000, 96
    centers = offset + rng.normal(0, 2, (K, d))
    lab = rng.integers(0, K, n).astype(np.int32)
    X = (centers[lab] + rng.normal(0, 0.5, (n, d))).astype(np.float32)
    C = (centers + rng.normal(0, 0.05, (K, d))).astype(np.float64)
    km = aakm.KMeans(dev(X), K, aakm.config())
    part = km.update_partials(dev(lab), dev(C)).cpu().numpy()
    km.close()
    E_ora = oracle.energy(X, C, lab)
    xn = np.sqrt((X.astype(np.float64) ** 2).sum(1).max()) * (1 + 1e-6)
    cm = np.sqrt(np.float32((C ** 2).sum(1).max()))
    eb = np.frexp(2.0 * (xn + cm) ** 2)[1]
    unit = 2.0 ** (eb - 51)                                    # 2^-30 / q
    bound = (n * d + 7 * K * d) * unit / 2 + 1e-13 * E_ora
    assert abs(part[-2] - E_ora) <= bound, (part[-2], E_ora, bound)


@pytest.mark.parametrize("cfg,N,K,bounded,comm", [("c4", 120_000, 128, True, False), ("c5", 100_000, 256, False, False),
                                                  ("c3", 90_000, 64, False, False), ("c5", 100_000, 256, False, True)])
def test_incremental_update_bitwise(cfg, N, K, bounded, comm, monkeypatch):
    """The incremental update (S(P^t) = S(P^{t-1}) + the moved rows, taken on the
    device when few rows move) is the full sort + segmented sums in exact
    integers: a whole Algorithm 1 run with it (every evaluation that qualifies)
    and without it (AAKM_DELTA_DIV=0) gives bitwise the same centroids, labels,
    energies and counts, and the trace shows it taken.  comm: through a real
    1-rank NCCL communicator, where S_ref is the rank's local partial and the
    allreduce reads it out of place (the multi-rank form)."""
    X, C0, c = make(cfg, N=N, K=K)
    out = {}
    monkeypatch.setenv("AAKM_UPD_PRIV", "0")                     # small K*d: the sort path (priv has no S_ref)
    for div in ("1", "0"):                                       # 1: moved rows <= n take it (always)
        monkeypatch.setenv("AAKM_DELTA_DIV", div)
        path = "tc16" if c.d in (64, 128) else "auto"
        km = aakm.KMeans(dev(X), c.K, aakm.config(m0=5, bounded=bounded, assign_path=path, max_iters=60,
                                                  comm_always=comm))
        C, lab, rep = km.run(dev(C0))
        out[div] = (C.cpu().numpy(), lab.cpu().numpy(), rep)
        ne, ni, moved = km.update_stats()
        if div == "1":
            assert ni > 0 and ni >= ne - 1 and moved > 0, (ne, ni, moved, rep)   # all but line 1
        else:
            assert ni == 0, (ne, ni)
        km.close()
    (Ca, la, ra), (Cb, lb, rb) = out["1"], out["0"]
    assert np.array_equal(Ca.view(np.int64), Cb.view(np.int64))
    assert np.array_equal(la, lb)
    for k in ("iters", "n_assign", "n_accepted", "n_rejected", "energy", "converged"):
        assert ra[k] == rb[k], (k, ra[k], rb[k])


@pytest.mark.parametrize("cfg,N,K,comm", [("c2", None, None, False), ("c2", 70_001, 100, False),
                                          ("c1", 80_000, 37, False), ("c2", None, None, True)])
def test_private_update_bitwise(cfg, N, K, comm, monkeypatch):
    """The one-kernel update of small K*d shards (shared-memory int32 sums of the
    same two-part fixed-point integers, <= 511 rows per block) against the
    label-sorted engine (sort + segmented sums, AAKM_UPD_PRIV=0): whole Algorithm 1
    runs bitwise equal (centroids, labels, energies, counts), ragged row counts,
    odd K, d = 2 and 16, and through a 1-rank NCCL communicator; and the partials
    of one G-evaluation equal the oracle's exact sums."""
    X, C0, c = make(cfg, N=N, K=K)
    out = {}
    for priv in ("1", "0"):
        monkeypatch.setenv("AAKM_UPD_PRIV", priv)
        km = aakm.KMeans(dev(X), c.K, aakm.config(m0=5, max_iters=200, comm_always=comm))
        C, lab, rep = km.run(dev(C0))
        out[priv] = (C.cpu().numpy(), lab.cpu().numpy(), rep)
        km.close()
    (Ca, la, ra), (Cb, lb, rb) = out["1"], out["0"]
    assert np.array_equal(Ca.view(np.int64), Cb.view(np.int64))
    assert np.array_equal(la, lb)
    for k in ("iters", "n_assign", "n_accepted", "n_rejected", "energy", "converged"):
        assert ra[k] == rb[k], (k, ra[k], rb[k])
    # one G-evaluation's sums against the oracle (Eq. 4: G = S / N, empty -> C row)
    monkeypatch.setenv("AAKM_UPD_PRIV", "1")
    km = aakm.KMeans(dev(X), c.K, aakm.config())
    lab0, _, _ = km.assign(dev(C0))
    G, n = km.update(lab0, dev(C0))
    G_ora, n_ora = oracle.update(X, lab0.cpu().numpy(), C0.astype(np.float64))
    assert np.array_equal(n.cpu().numpy(), n_ora)
    np.testing.assert_allclose(G.cpu().numpy(), G_ora, rtol=1e-12, atol=1e-12)
    km.close()
