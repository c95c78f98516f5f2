"""-m gpu: BASELINE.json's full-size configs in the launch configuration bench.py
times (auto engine, CTA pairs, graph-free aa_step), checked against the CPU
oracle where it can afford it:
  * assignment: a seeded 1 % row sample (at least 20 000 rows)
    decided by the oracle one row at a time (north-star tie rule), plus label
    range / counts properties for all rows;
  * energy and update: the oracle's full O(N d) sums over every row (exact fp64);
  * one Algorithm 1 pass after line 1: the exported C^{t+1} is finite and the
    accepted / rejected energies obey the guard.
c1 and c2 are small enough for the element-wise parity tests of test_gpu_parity."""
import numpy as np
import pytest

import oracle
from gpu_helpers import check_assign, dev, g_close, require_gpu, torch
from paper_1805_10638_b200 import aakm, synthetic

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu():
    require_gpu()


@pytest.mark.parametrize("cfg,path", [("c3", "auto"), ("c4", "auto"), ("c5", "auto"), ("c5", "tc")])
def test_full_size_sampled(cfg, path):
    X, C0, c = synthetic.make(cfg, seed=0)
    Xd = dev(X)
    km = aakm.KMeans(Xd, c.K, aakm.config(m0=c.m0, assign_path=path))
    km.aa_step(dev(C0), info=False)                       # Algorithm 1 line 1
    info = km.aa_step()                                    # one loop pass
    assert info["t"] == 1 and np.isfinite(info["energy"])
    s = km.state_export()
    C = s["C"]                                             # C^{t+1}
    assert np.isfinite(C).all()
    lab, E, _ = km.assign(dev(C))
    lab = lab.cpu().numpy()
    assert lab.min() >= 0 and lab.max() < c.K
    rng = np.random.default_rng(2024)
    rows = np.sort(rng.choice(c.N, max(20_000, c.N // 100), replace=False))
    check_assign(X[rows], C, lab[rows], msg=f"{cfg}/{path} sampled rows")
    E_ora = oracle.energy(X, C.astype(np.float64), lab)   # every row, fp64
    assert abs(E - E_ora) <= 1e-6 * E_ora, (E, E_ora)
    G, cnt = km.update(dev(lab), dev(C))
    G_ora, cnt_ora = oracle.update(X, lab, C.astype(np.float64))
    np.testing.assert_array_equal(cnt.cpu().numpy(), cnt_ora)
    assert int(cnt_ora.sum()) == c.N
    err, ok = g_close(G.cpu().numpy(), G_ora)
    assert ok.all(), f"{cfg}: G rel err {err}"
    km.close()
