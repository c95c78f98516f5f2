"""-m gpu: f4, the combine fused into the update's flushes (cfg.fused_comm, comm.cu)
on a real 1-rank communicator (cfg.comm_always).  The packed [S|N|E|changed]
vectors live in an NCCL symmetric window; the flushes add into every replica
(multimem through the NVLS multicast address, or system-scope reds to each LSA
peer), with the "zeroed" / "flushed" device barriers around them and no
allreduce launch.  The results must be bitwise those of the plain path (exact
integer sums) -- for the graph-captured kmeans_run and for eager passes -- in
both transport modes (AAKM_FUSED_MODE=2 forces the unicast one)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from gpu_helpers import dev, make, require_gpu, torch
from paper_1805_10638_b200 import aakm

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(autouse=True)
def _gpu():
    require_gpu()


CASES = [("c1", None, None, False), ("c2", None, None, False), ("c5", 70_000, 256, False),
         ("c5", 70_000, 256, True), ("c3", 40_000, 64, False)]


def _compare(cfg, N, K, bounded):
    X, C0, c = make(cfg, N=N, K=K)
    Xd = dev(X)
    a = aakm.KMeans(Xd, c.K, aakm.config(m0=5, bounded=bounded, max_iters=300))
    b = aakm.KMeans(Xd, c.K, aakm.config(m0=5, bounded=bounded, max_iters=300, comm_always=True, fused_comm=True))
    mode, lsa = b.comm_info()
    assert mode in (1, 2) and lsa == 1, (mode, lsa)
    assert a.comm_info()[0] == -1
    Ca, la, ra = a.run(dev(C0))
    Cb, lb, rb = b.run(dev(C0))
    assert np.array_equal(Ca.cpu().numpy().view(np.uint64), Cb.cpu().numpy().view(np.uint64))
    assert torch.equal(la, lb)
    for k in ("iters", "n_assign", "n_accepted", "n_rejected", "converged", "m_final", "energy"):
        assert ra[k] == rb[k], (k, ra, rb)
    a.aa_step(dev(C0)); b.aa_step(dev(C0))
    for _ in range(4):
        ia, ib = a.aa_step(), b.aa_step()
        assert ia == ib, (ia, ib)
    a.close(); b.close()
    return mode


@pytest.mark.parametrize("cfg,N,K,bounded", CASES)
def test_fused_combine_is_bitwise_identical(cfg, N, K, bounded):
    _compare(cfg, N, K, bounded)


def test_fused_combine_unicast_mode_subprocess():
    code = r"""
import sys
sys.path.insert(0, %r); sys.path.insert(0, %r)
import test_gpu_fused as t
for c in t.CASES[:3]:
    assert t._compare(*c) == 2
print("ok")
""" % (ROOT, os.path.join(ROOT, "tests"))
    env = dict(os.environ, AAKM_FUSED_MODE="2")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]


def test_fused_needs_a_communicator():
    X, C0, c = make("c1")
    with pytest.raises(aakm.AAKMError):
        aakm.KMeans(dev(X), c.K, aakm.config(fused_comm=True))
