"""CPU oracle for Anderson-accelerated Lloyd K-Means (arXiv 1805.10638).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_1805_10638_b200`` never imports it and
the two share no code.  See ``oracle/aakm_oracle.c`` for the algorithm and
its citations, and DESIGN.md §3 for the pins.
"""
from .oracle import (  # noqa: F401
    build, lib, assign, best2, energy, update, ls_solve, adjust_m, sqdist,
    OracleConfig, AAState, run, lloyd, seed_pp, seed_scale, SeedError,
)
