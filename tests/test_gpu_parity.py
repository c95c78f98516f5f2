"""-m gpu: the CUDA path (through the C ABI) against the CPU oracle on the same
seeded inputs.  Tolerances are the north_star's (BASELINE.json):
  * labels bit-exact except where the oracle's best-vs-chosen gap <= 1e-5 rel;
  * centroids <= 1e-5 relative (per element, floor rms(G)); energy <= 1e-6 rel;
  * end-to-end: same iteration count, final energy within 1e-4 relative on the
    well-separated configs (c1, c2, c4).
"""
import numpy as np
import pytest

import oracle
from gpu_helpers import check_assign, dev, g_close, make, require_gpu, torch
from paper_1805_10638_b200 import aakm

pytestmark = pytest.mark.gpu

# (cfg, N, K) small variants that still span many tiles and a ragged tail
CASES = [("c1", None, None), ("c2", None, None), ("c3", 30_011, None), ("c4", 8_003, None), ("c5", 8_009, None)]


@pytest.fixture(autouse=True)
def _gpu():
    require_gpu()


def handle(X, K, path="auto", **kw):
    return aakm.KMeans(dev(X), K, aakm.config(assign_path=path, **kw))


def tc16_ok(d):
    return d in (64, 128)


@pytest.mark.parametrize("cfg,N,K", CASES)
@pytest.mark.parametrize("path", ["auto", "simt", "tc", "tc16"])
def test_assign_parity(cfg, N, K, path):
    X, C0, c = make(cfg, N=N, K=K)
    if path == "tc" and c.d % 32:
        pytest.skip("3xTF32 engine needs d % 32 == 0")
    if path == "tc16" and c.d not in (64, 128):
        pytest.skip("2xFP16 engine needs d in {64, 128}")
    km = handle(X, c.K, path)
    rng = np.random.default_rng(1)
    prev = rng.integers(0, c.K, size=c.N).astype(np.int32)
    # C^0 (samples: fp32 values) and a perturbed fp64 C (the Algorithm 1 state is fp64)
    for C in (C0.astype(np.float64), C0 + rng.normal(0, 0.05, C0.shape)):
        lab, E, ch = km.assign(dev(C), dev(prev))
        lab = lab.cpu().numpy()
        lab_ora, ndiff = check_assign(X, C, lab, msg=f"{cfg}/{path}")
        E_ora = oracle.energy(X, C.astype(np.float64), lab)
        assert abs(E - E_ora) <= 1e-6 * E_ora
        assert ch == int((lab != prev).sum())
    km.close()


@pytest.mark.parametrize("cfg,N,K", CASES)
def test_update_parity(cfg, N, K):
    X, C0, c = make(cfg, N=N, K=K)
    km = handle(X, c.K)
    lab = oracle.assign(X, C0.astype(np.float64))
    lab[:7] = 0                                      # make sure some structure changes
    Cprev = C0.copy()
    Cprev[-1] += 1e4                                 # far away: cluster K-1 ends up empty
    lab[lab == c.K - 1] = 0
    G, cnt = km.update(dev(lab), dev(Cprev))
    G_ora, cnt_ora = oracle.update(X, lab, Cprev.astype(np.float64))
    np.testing.assert_array_equal(cnt.cpu().numpy(), cnt_ora)
    err, ok = g_close(G.cpu().numpy(), G_ora)
    assert ok.all(), f"max rel err {err}"
    np.testing.assert_array_equal(G.cpu().numpy()[-1], Cprev[-1])   # empty cluster keeps C_prev (R-A15)
    km.close()


def test_update_rejects_bad_labels():
    X, C0, c = make("c1")
    km = handle(X, c.K)
    lab = np.zeros(c.N, np.int32); lab[5] = c.K
    with pytest.raises(aakm.AAKMError):
        km.update(dev(lab), dev(C0))
    km.close()


def test_assign_edge_cases():
    # SPEC.md:99-101 worked examples through the GPU path
    X = np.array([[0], [1], [4], [5]], np.float32)
    km = handle(X, 2)
    lab, E, _ = km.assign(dev(np.array([[0], [5]], np.float32)))
    assert lab.cpu().tolist() == [0, 0, 1, 1] and E == 2.0
    km.close()
    km = handle(np.array([[2.0]], np.float32), 1)
    lab, E, _ = km.assign(dev(np.array([[1.0]], np.float32)))
    assert lab.cpu().tolist() == [0] and E == 1.0
    km.close()
    X = np.array([[2.0], [2.0], [0.5]], np.float32)               # exact tie x=2 between 1 and 3 -> index 0
    km = handle(X, 2)
    lab, _, _ = km.assign(dev(np.array([[1.0], [3.0]], np.float32)))
    assert lab.cpu().tolist() == [0, 0, 0]
    km.close()


@pytest.mark.parametrize("cfg", ["c2", "c4", "c5"])
def test_assign_duplicate_centroids_and_self(cfg):
    # duplicated centroid rows are exact ties (lowest index wins); rows that ARE
    # centroids have d_best = 0; K = 1 degenerates to all-zero labels.
    X, C0, c = make(cfg, N=5001)
    C = C0.copy()
    C[7] = C[3]
    km = handle(X, c.K)
    lab, E, _ = km.assign(dev(C))
    lab = lab.cpu().numpy()
    lab_ora, _ = check_assign(X, C, lab)
    assert not np.any(lab == 7)
    np.testing.assert_array_equal(lab, lab_ora)
    km.close()
    km = handle(X, 1)
    lab, E, _ = km.assign(dev(C[:1]))
    assert int(lab.abs().sum()) == 0
    assert abs(E - oracle.energy(X, C[:1].astype(np.float64), np.zeros(len(X), np.int32))) <= 1e-6 * E
    km.close()


@pytest.mark.parametrize("n", [1, 31, 257, 1025])
def test_ragged_small_n(n):
    X, C0, c = make("c4", N=max(n, 16), K=16)
    X = X[:n]
    C = C0[: min(16, n)]
    km = handle(X, len(C))
    lab, E, _ = km.assign(dev(C))
    check_assign(X, C, lab.cpu().numpy())
    km.close()


def _lockstep(cfg, N=None, K=None, seed=0, m0=5, max_passes=400, path="auto", dynamic_m=True):
    X, C0, c = make(cfg, seed=seed, N=N, K=K)
    km = handle(X, c.K, path, m0=m0, dynamic_m=dynamic_m)
    info0 = km.aa_step(dev(C0))
    ora = oracle.AAState(X, oracle.OracleConfig(m0=m0, dynamic_m=dynamic_m))
    ora.init(C0.astype(np.float64))
    s = km.state_export()
    err, ok = g_close(s["C"], ora.C)
    assert ok.all(), f"init C^1 rel err {err}"
    assert info0["t"] == 0
    npass = 0
    for _ in range(max_passes):
        s = km.state_export()
        if s["done"]:
            break
        ora.load(C=s["C"], fallback=s["fallback"], Ghist=s["Ghist"], Fhist=s["Fhist"],
                 labels_prev=s["labels_prev"], E1=s["E1"], E2=s["E2"], m=s["m"], lloyd=s["lloyd"], t=s["t"])
        rc = ora.step()
        oi = ora.info()
        gi = km.aa_step()
        npass += 1
        tag = f"{cfg} pass t={s['t']}"
        assert gi["converged"] == (rc == 1), tag
        assert gi["rejected"] == oi["rejected"], tag
        assert abs(gi["energy_cand"] - oi["E_cand"]) <= 1e-6 * oi["E_cand"], tag
        assert abs(gi["energy"] - oi["E"]) <= 1e-6 * oi["E"], tag
        assert gi["changed"] == oi["changed"], tag
        if rc == 1:
            break
        assert gi["accepted"] == oi["accepted"] and gi["m"] == oi["m"] and gi["m_t"] == oi["m_t"], tag
        s2 = km.state_export()
        err, okc = g_close(s2["C"], ora.C)
        assert okc.all(), f"{tag}: C^(t+1) rel err {err}"
    km.close()
    return npass


@pytest.mark.parametrize("cfg,N,K,seed", [("c1", None, None, 0), ("c1", None, None, 3), ("c2", None, None, 0),
                                          ("c3", 20_000, 64, 0), ("c4", 6_000, 128, 0), ("c5", 4_000, 256, 0)])
def test_aa_step_lockstep(cfg, N, K, seed):
    n = _lockstep(cfg, N, K, seed)
    assert n >= 2


@pytest.mark.parametrize("cfg,N,K", [("c4", 6_000, 128), ("c5", 4_000, 256)])
def test_aa_step_lockstep_tc16(cfg, N, K):
    assert _lockstep(cfg, N, K, 0, path="tc16") >= 2


@pytest.mark.parametrize("cfg,N,K,seed,path", [("c1", None, None, s, "auto") for s in range(5)] +
                         [("c2", None, None, 0, "auto"), ("c2", None, None, 1, "auto"), ("c4", 8_000, 256, 0, "tc"),
                          ("c4", 8_000, 256, 0, "tc16"), ("c4", 20_000, 1024, 1, "tc16")])
def test_end_to_end_parity(cfg, N, K, seed, path):
    X, C0, c = make(cfg, seed=seed, N=N, K=K)
    km = handle(X, c.K, path, m0=5)
    C, lab, rep = km.run(dev(C0))
    ref = oracle.run(X, C0.astype(np.float64), oracle.OracleConfig(m0=5))
    assert rep["converged"] and ref["converged"]
    assert rep["iters"] == ref["iters"], (rep, {k: v for k, v in ref.items() if k not in ("C", "labels", "trace")})
    assert abs(rep["energy"] - ref["energy"]) <= 1e-4 * ref["energy"]
    assert rep["n_assign"] == rep["iters"] + rep["n_rejected"]
    # the returned C is a fixed point: it is the mean of its own partition
    G, _ = km.update(lab, C)
    err, ok = g_close(G.cpu().numpy(), C.cpu().numpy())
    assert ok.all(), err
    err, ok = g_close(C.cpu().numpy(), ref["C"])
    assert ok.all(), f"final C vs oracle: {err}"
    km.close()


@pytest.mark.parametrize("cfg,N,K,m0", [("c1", None, None, 2), ("c1", None, None, 5), ("c2", None, None, 2),
                                        ("c2", None, None, 5), ("c4", 8_000, 256, 2)])
def test_fixed_m_end_to_end(cfg, N, K, m0):
    # Table 2's "Fixed m" columns: dynamic_m = 0, m = m0 throughout
    X, C0, c = make(cfg, N=N, K=K)
    km = handle(X, c.K, m0=m0, dynamic_m=False)
    C, lab, rep = km.run(dev(C0))
    ref = oracle.run(X, C0.astype(np.float64), oracle.OracleConfig(m0=m0, dynamic_m=False))
    assert rep["converged"] and ref["converged"]
    assert rep["m_final"] == m0 == ref["m_final"]
    assert rep["iters"] == ref["iters"] and rep["n_rejected"] == ref["rejected"]
    assert abs(rep["energy"] - ref["energy"]) <= 1e-4 * ref["energy"]
    km.close()


@pytest.mark.parametrize("cfg,N,K,m0", [("c2", None, None, 2), ("c4", 6_000, 128, 5)])
def test_fixed_m_lockstep(cfg, N, K, m0):
    assert _lockstep(cfg, N, K, 0, m0=m0, dynamic_m=False) >= 2


@pytest.mark.parametrize("cfg,N,K", [("c1", None, None), ("c2", None, None), ("c4", 6_000, 128)])
def test_m0_is_lloyd_on_gpu(cfg, N, K):
    X, C0, c = make(cfg, N=N, K=K)
    km = handle(X, c.K, m0=0, dynamic_m=False)
    C, lab, rep = km.run(dev(C0))
    ref = oracle.lloyd(X, C0.astype(np.float64))
    assert rep["n_accepted"] == 0 and rep["n_rejected"] == 0
    assert rep["iters"] == ref["iters"]
    assert abs(rep["energy"] - ref["energy"]) <= 1e-6 * ref["energy"]
    km.close()


@pytest.mark.parametrize("max_iters", [1, 3, 8])
def test_max_iters_reported_not_error(max_iters):
    # stopping at the cap returns C^{t+1} and the labels P^t of the last pass, as the oracle does
    X, C0, c = make("c2")
    km = handle(X, c.K, max_iters=max_iters)
    C, lab, rep = km.run(dev(C0))
    ref = oracle.run(X, C0.astype(np.float64), oracle.OracleConfig(m0=5, max_iters=max_iters))
    assert rep["converged"] == 0 and not ref["converged"]
    assert rep["iters"] == ref["iters"] == max_iters + 1
    np.testing.assert_array_equal(lab.cpu().numpy(), ref["labels"])
    err, ok = g_close(C.cpu().numpy(), ref["C"])
    assert ok.all(), err
    C2, lab2 = km.centroids()                         # the same buffers through get_centroids
    np.testing.assert_array_equal(lab2.cpu().numpy(), lab.cpu().numpy())
    np.testing.assert_array_equal(C2.cpu().numpy(), C.cpu().numpy())
    st = km.state_export()                            # a finished state exports its final labels
    assert st["done"] == 1
    np.testing.assert_array_equal(st["labels_prev"], ref["labels"])
    km.close()


def test_accepted_energies_monotone_on_gpu():
    X, C0, c = make("c3", N=50_000)
    km = handle(X, c.K)
    km.aa_step(dev(C0))
    Es = []
    for _ in range(60):
        gi = km.aa_step()
        Es.append(gi["energy"])
        if gi["converged"]:
            break
    assert all(b <= a * (1 + 1e-12) for a, b in zip(Es, Es[1:]))
    km.close()


@pytest.mark.parametrize("cfg,N,K,m0", [("c1", None, None, 5), ("c2", None, None, 2)])
def test_trace_export_matches_oracle_trace(cfg, N, K, m0):
    # kmeans_trace_export: one record per loop pass of a kmeans_run, against the oracle's own trace
    X, C0, c = make(cfg, N=N, K=K)
    km = handle(X, c.K, m0=m0)
    _, _, rep = km.run(dev(C0))
    tr = km.trace()
    ref = oracle.run(X, C0.astype(np.float64), oracle.OracleConfig(m0=m0), trace=True)
    assert len(tr) == len(ref["trace"]) == rep["iters"] - 1
    for g, o in zip(tr, ref["trace"]):
        tag = f"{cfg} t={o['t']}"
        assert g["t"] == o["t"] and g["m"] == o["m"] and g["changed"] == o["changed"], (tag, g, o)
        assert g["accepted"] == o["accepted"] and g["rejected"] == o["rejected"], (tag, g, o)
        assert abs(g["energy"] - o["E"]) <= 1e-6 * o["E"], (tag, g, o)
        assert abs(g["energy_cand"] - o["E_cand"]) <= 1e-6 * o["E_cand"], (tag, g, o)
    assert tr[-1]["converged"] == 1
    km.close()
