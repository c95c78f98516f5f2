"""-m "not gpu": the seeded generators are deterministic (same bytes every call,
every thread schedule) and the shards equal the full draw's rows."""
import hashlib

import numpy as np

from paper_1805_10638_b200 import synthetic


def test_c4_full_draw_is_repeatable_and_sharded_consistently():
    # c4's chunk threads multiply with BLAS; unserialised, concurrent calls corrupted rows
    X1, C1, c = synthetic.make("c4")
    X2, C2, _ = synthetic.make("c4", threads=16)
    assert hashlib.md5(X1.tobytes()).digest() == hashlib.md5(X2.tobytes()).digest()
    assert np.array_equal(C1, C2)
    lo, hi = synthetic.shard_bounds(c.N, 1, 3)
    Xs, Cs, _ = synthetic.make_shard("c4", 1, 3)
    assert np.array_equal(Xs, X1[lo:hi]) and np.array_equal(Cs, C1)


def test_seed_uniforms_are_fixed():
    u = synthetic.seed_uniforms("c5", 64)
    assert np.array_equal(u, synthetic.seed_uniforms("c5", 64))
    assert u.min() >= 0.0 and u.max() < 1.0
