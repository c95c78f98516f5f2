"""Shared helpers for the -m gpu parity tests (CUDA path vs the CPU oracle)."""
import numpy as np
import pytest

import oracle
from paper_1805_10638_b200 import synthetic

torch = pytest.importorskip("torch")


def require_gpu():
    # GPU tests must fail loudly (not skip) on a box without CUDA: the driver runs -m gpu on a B200.
    assert torch.cuda.is_available(), "-m gpu tests need a CUDA device"


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a)).cuda()


def make(cfg, seed=0, N=None, K=None):
    X, C0, c = synthetic.make(cfg, seed=seed, N=N, K=K)
    return X, C0, c


def check_assign(X, C, lab_gpu, rel=1e-5, msg=""):
    """North-star rule: labels bit-exact except where the oracle's best-vs-chosen
    squared-distance gap is <= 1e-5 relative (floor for d_best = 0)."""
    lab_gpu = np.asarray(lab_gpu)
    lab_ora = oracle.assign(X, C.astype(np.float64))
    diff = np.nonzero(lab_gpu != lab_ora)[0]
    if len(diff):
        Xd = X[diff].astype(np.float64)
        Cd = C.astype(np.float64)
        dch = ((Xd - Cd[lab_gpu[diff]]) ** 2).sum(1)
        dbe = ((Xd - Cd[lab_ora[diff]]) ** 2).sum(1)
        floor = 1e-12 * ((Xd ** 2).sum(1) + (Cd[lab_ora[diff]] ** 2).sum(1))
        bad = (dch - dbe) > np.maximum(rel * dbe, floor)
        assert not bad.any(), f"{msg}: {bad.sum()} labels outside the tie band, rows {diff[bad][:10]}"
    return lab_ora, len(diff)


def g_close(G_gpu, G_ora, rel=1e-5):
    G_gpu = np.asarray(G_gpu, np.float64); G_ora = np.asarray(G_ora, np.float64)
    scale = np.maximum(np.abs(G_ora), np.sqrt(np.mean(G_ora ** 2)))
    err = np.abs(G_gpu - G_ora) / scale
    return float(err.max()), err <= rel
