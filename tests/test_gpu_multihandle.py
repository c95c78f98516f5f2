"""-m gpu: data-parallel decomposition through the C ABI on one GPU.  Two
handles own the two row halves of a shard (as two ranks would); their
unreduced kmeans_update_partials summed on the host must equal the
one-handle partials and the oracle's full-data update/energy/changed.
(NCCL refuses two ranks on one GPU, and this build has one GPU, so the
allreduce itself is exercised only on real multi-GPU runs.)"""
import numpy as np
import pytest

import oracle
from gpu_helpers import dev, make, require_gpu, torch
from paper_1805_10638_b200 import aakm, synthetic

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,N", [("c1", None), ("c2", None), ("c3", 40_000), ("c5", 30_000)])
@pytest.mark.parametrize("world", [2, 3])
def test_partials_sum_over_shards(cfg, N, world):
    require_gpu()
    X, C0, c = make(cfg, N=N)
    C = C0.astype(np.float64) + 0.01
    prev = oracle.assign(X, C0.astype(np.float64))
    lab = oracle.assign(X, C.astype(np.float64))
    K, d = C.shape
    tot = np.zeros(K * d + K + 2)
    for r in range(world):
        lo, hi = synthetic.shard_bounds(c.N, r, world)
        km = aakm.KMeans(dev(X[lo:hi]), K, aakm.config(), n_global=c.N)
        tot += km.update_partials(dev(lab[lo:hi]), dev(C), labels_prev=dev(prev[lo:hi])).cpu().numpy()
        km.close()
    km = aakm.KMeans(dev(X), K, aakm.config())
    one = km.update_partials(dev(lab), dev(C), labels_prev=dev(prev)).cpu().numpy()
    km.close()
    np.testing.assert_allclose(tot[:K * d], one[:K * d], rtol=1e-12, atol=1e-9)
    np.testing.assert_array_equal(tot[K * d:K * d + K], one[K * d:K * d + K])
    assert tot[-1] == one[-1] == float((lab != prev).sum())
    E_ora = oracle.energy(X, C.astype(np.float64), lab)
    assert abs(tot[-2] - E_ora) <= 1e-9 * E_ora and abs(one[-2] - E_ora) <= 1e-9 * E_ora
    G_ora, cnt = oracle.update(X, lab, C.astype(np.float64))
    np.testing.assert_array_equal(tot[K * d:K * d + K], cnt)
    S = tot[:K * d].reshape(K, d)
    G = np.where(cnt[:, None] > 0, S / np.maximum(cnt, 1)[:, None], C)
    np.testing.assert_allclose(G, G_ora, rtol=1e-12, atol=1e-12)
