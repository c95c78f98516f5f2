"""-m gpu: the NCCL data plane on one GPU (cfg.comm_always = 1: a real 1-rank
communicator).  Every allreduce of the path -- the create-time max of the X
statistics, the per-G-evaluation int64 allreduce of the packed exact partials
(eager and captured in the kmeans_run CUDA graph), the three K-Means++
exchanges per center -- runs through NCCL, and the results must be bitwise
those of the communicator-free path (the allreduced vector is integer, so a
1-rank sum is the identity, `north_star` row a7)."""
import numpy as np
import pytest

import oracle
from gpu_helpers import check_assign, dev, make, require_gpu, torch
from paper_1805_10638_b200 import aakm, synthetic

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu():
    require_gpu()


def _pair(X, K, **kw):
    Xd = dev(X)
    return (aakm.KMeans(Xd, K, aakm.config(**kw)), aakm.KMeans(Xd, K, aakm.config(comm_always=True, **kw)))


@pytest.mark.parametrize("cfg,N,K,bounded", [("c1", None, None, False), ("c2", None, None, False),
                                             ("c5", 70_000, 256, False), ("c5", 70_000, 256, True),
                                             ("c3", 40_000, 64, False)])
def test_run_through_nccl_is_bitwise_identical(cfg, N, K, bounded):
    X, C0, c = make(cfg, N=N, K=K)
    a, b = _pair(X, c.K, m0=5, bounded=bounded, max_iters=300)
    Ca, la, ra = a.run(dev(C0))
    Cb, lb, rb = b.run(dev(C0))                     # graph-captured ncclAllReduce per G-evaluation
    if c.N >= 65_536 and c.K * c.d > 4096:         # sorted engine, not the one-kernel small-K*d update:
        assert b.update_stats()[1] > 0              # the incremental update ran through the communicator
    assert np.array_equal(Ca.cpu().numpy().view(np.uint64), Cb.cpu().numpy().view(np.uint64))
    assert torch.equal(la, lb)
    for k in ("iters", "n_assign", "n_accepted", "n_rejected", "converged", "m_final", "energy"):
        assert ra[k] == rb[k], (k, ra, rb)
    # eager passes (kmeans_aa_step) through the communicator as well
    a.aa_step(dev(C0)); b.aa_step(dev(C0))
    for _ in range(5):
        ia, ib = a.aa_step(), b.aa_step()
        assert ia == ib, (ia, ib)
    a.close(); b.close()


def test_api_calls_through_nccl():
    X, C0, c = make("c5", N=70_000, K=256)
    a, b = _pair(X, c.K)
    C = C0 + np.random.default_rng(3).normal(0, 0.02, C0.shape)
    la, Ea, _ = a.assign(dev(C))
    lb, Eb, _ = b.assign(dev(C))
    assert torch.equal(la, lb) and Ea == Eb
    check_assign(X, C, lb.cpu().numpy())
    Ga, na = a.update(la, dev(C))
    Gb, nb = b.update(lb, dev(C))
    assert torch.equal(Ga, Gb) and torch.equal(na, nb)
    G_ora, _ = oracle.update(X, lb.cpu().numpy(), C)
    np.testing.assert_allclose(Gb.cpu().numpy(), G_ora, rtol=1e-12, atol=1e-12)
    a.close(); b.close()


def test_seed_pp_through_nccl():
    X, _, c = make("c4", N=30_000, K=64)
    a, b = _pair(X, c.K)
    u = synthetic.seed_uniforms("c4", c.K)
    Ca, ia = a.seed_pp(u)
    Cb, ib = b.seed_pp(u)                           # max / totals / row exchange through NCCL
    assert np.array_equal(ia, ib) and torch.equal(Ca, Cb)
    assert np.array_equal(ib, oracle.seed_pp(X, c.K, u))
    a.close(); b.close()
