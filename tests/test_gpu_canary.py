"""-m gpu: checked-workspace runs (compute-sanitizer is closed on the GPU pool).
With AAKM_WS_CANARY=1 every region of the workspace carve is followed by a
256-byte canary; after runs of every engine -- SIMT (c1, c2, odd d), 3xTF32,
2xFP16 dense and bounded, the candidate pass, the label-sorted and the atomic
update, K-Means++ seeding, ragged K and tiny n -- no canary byte may change
(an out-of-bounds write past any region of the workspace would)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
from paper_1805_10638_b200 import aakm, synthetic

def check(km, tag):
    bad, n = km.check_canaries()
    assert n > 10 and bad == 0, (tag, bad, n)

def run(X, C0, K, tag, **kw):
    km = aakm.KMeans(torch.from_numpy(np.ascontiguousarray(X)).cuda(), K, aakm.config(m0=5, **kw))
    C, lab, rep = km.run(torch.from_numpy(np.ascontiguousarray(C0)).cuda())
    lab2, E, ch = km.assign(C, labels_prev=lab)
    G, cnt = km.update(lab2, C)
    km.aa_step(torch.from_numpy(np.ascontiguousarray(C0)).cuda())
    for _ in range(3):
        km.aa_step()
    check(km, tag)
    return km

for cfg, N, K, kw in [("c1", None, None, {}), ("c2", 4000, None, {}), ("c3", 70000, 64, dict(assign_path="tc", max_iters=8)),
                      ("c5", 70000, 256, dict(assign_path="tc16", max_iters=8)),
                      ("c5", 70000, 256, dict(assign_path="tc16", bounded=True, max_iters=8)),
                      ("c4", 20000, 300, dict(max_iters=8)), ("c5", 70000, 129, dict(assign_path="tc", max_iters=5))]:
    X, C0, c = synthetic.make(cfg, N=N, K=K)
    km = run(X, C0, c.K, f"{cfg}/{kw}", **kw)
    km.close()
X, C0, c = synthetic.make("c4", N=20000, K=32)
km = aakm.KMeans(torch.from_numpy(X).cuda(), c.K, aakm.config())
km.seed_pp(synthetic.seed_uniforms("c4", c.K))
check(km, "seed")
km.close()
rng = np.random.default_rng(5)
for d, n, K in [(3, 70000, 37), (33, 5000, 7), (64, 1, 1), (128, 31, 5)]:
    X = rng.normal(0, 2, (n, d)).astype(np.float32)
    km = run(X, X[:K].astype(np.float64), K, f"d={d} n={n}", max_iters=6)
    km.close()
print("canaries ok")
""" % ROOT


def test_workspace_canaries_intact():
    env = dict(os.environ, AAKM_WS_CANARY="1")
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "canaries ok" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
