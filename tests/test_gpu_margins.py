"""-m gpu: measured exactness margins of the assignment engines (row a3's
premise).  Every engine flags a row as a near tie when its computed top-2 gap
b2 - b1 is within tau, and tau is twice a rigorous per-value error bound
(DESIGN.md §5.3).  kmeans_debug_scores exports (b1, b2, tau) per row before the
refine; here the exact counterparts are formed in fp64 and

    r = max(|b1 - e1|, |b2 - e2|) / tau   (e1 <= e2: the two smallest exact values)

must stay <= 1/2 on every sampled row (|min a - min e| <= max |a - e|, the same
for the second order statistic).  Inputs: BASELINE configs at full size (1 %
row samples), plus adversarial ones: large ||x|| against small distances (the
c4 cancellation, 1000x worse), and coordinates spanning ten decades (the fp16
subnormal floors of the 2xFP16 split).  The distribution is appended to
gpurun_out/margins.jsonl (profiles/r02_margins.jsonl keeps a copy)."""
import json
import os

import numpy as np
import pytest

from gpu_helpers import dev, require_gpu, torch
from paper_1805_10638_b200 import aakm, synthetic

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(autouse=True)
def _gpu():
    require_gpu()


def _exact_top2(X, C, kind, unit):
    """The engine's value of every centroid, exactly (fp64; the expansion's
    rounding, ~1e-16 of ||x||^2 + ||c||^2, is far below every tau)."""
    Xd = X.astype(np.float64)
    xn = (Xd ** 2).sum(1)
    cn = (C ** 2).sum(1)
    e1 = np.empty(len(X)); e2 = np.empty(len(X))
    for a in range(0, len(X), 8192):
        s = cn[None, :] - 2.0 * Xd[a:a + 8192] @ C.T               # ||c||^2 - 2 x.c
        if kind == 0:
            v = 0.5 * s                                             # 3xTF32: ||c||^2/2 - x.c
        elif kind == 1:
            v = unit * (s + xn[a:a + 8192, None]) + 6.0             # 2xFP16 window: U ||x - c||^2 + 6
        else:
            v = s                                                   # SIMT: ||c||^2 - 2 x.c
        p = np.partition(v, 1, axis=1)[:, :2]
        e1[a:a + 8192] = p[:, 0]; e2[a:a + 8192] = p[:, 1]
    return e1, e2


def _measure(name, X, C, path, rows):
    km = aakm.KMeans(dev(X), C.shape[0], aakm.config(assign_path=path))
    out, kind, unit = km.debug_scores(C)
    eng = km.path
    km.close()
    out = out.cpu().numpy()[rows].astype(np.float64)
    e1, e2 = _exact_top2(X[rows], C, kind, unit)
    b1, b2, tau = out[:, 0], out[:, 1], out[:, 2]
    r = np.maximum(np.abs(b1 - e1), np.abs(b2 - e2)) / tau
    rec = {"case": name, "engine": eng, "rows": int(len(rows)), "N": int(len(X)), "d": int(X.shape[1]),
           "K": int(C.shape[0]), "r_max": float(r.max()), "r_p999": float(np.quantile(r, 0.999)),
           "r_p50": float(np.median(r)), "flag_frac": float(np.mean(b2 - b1 <= tau))}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "margins.jsonl"), "a") as f:
        f.write(json.dumps(rec) + "\n")
    assert np.isfinite(r).all() and r.max() <= 0.5, rec
    return rec


@pytest.mark.parametrize("cfg,path", [("c1", "auto"), ("c2", "auto"), ("c3", "auto"), ("c4", "auto"),
                                      ("c5", "auto"), ("c4", "tc"), ("c5", "tc")])
def test_margins_full_size(cfg, path):
    X, C0, c = synthetic.make(cfg, seed=0)
    rng = np.random.default_rng(7)
    # a mid-run-like C: C^0 plus small moves (the bound must hold for any C)
    C = C0.astype(np.float64) + rng.normal(0, 0.01 * float(np.std(C0)), C0.shape)
    rows = np.sort(rng.choice(c.N, min(c.N, max(20_000, c.N // 100)), replace=False))
    _measure(f"{cfg}-full", X, C, path, rows)


@pytest.mark.parametrize("path,d", [("tc16", 128), ("tc", 128), ("simt", 16), ("tc16", 64)])
def test_margins_large_norm(path, d):
    # clusters of radius ~1 around points at distance ~1e3 from the origin: ||x||^2 / d_best ~ 1e6
    rng = np.random.default_rng(d)
    n, K = 60_000, 256
    mu = 1000.0 + rng.normal(0, 3, (K, d))
    X = (mu[rng.integers(0, K, n)] + rng.normal(0, 0.3, (n, d))).astype(np.float32)
    C = mu + rng.normal(0, 0.05, mu.shape)
    _measure(f"large-norm-{path}-d{d}", X, C, path, np.arange(0, n, 3))


@pytest.mark.parametrize("path,d", [("tc16", 64), ("tc", 32), ("simt", 8)])
def test_margins_wide_range(path, d):
    # coordinates with magnitudes spanning 1e-8 .. 1e2 and random signs
    rng = np.random.default_rng(100 + d)
    n, K = 50_000, 300
    mag = 10.0 ** rng.uniform(-8, 2, (n, d))
    X = (mag * rng.choice([-1.0, 1.0], (n, d))).astype(np.float32)
    C = X[rng.choice(n, K, replace=False)].astype(np.float64) * (1 + rng.normal(0, 1e-3, (K, d)))
    _measure(f"wide-range-{path}-d{d}", X, C, path, np.arange(0, n, 2))
