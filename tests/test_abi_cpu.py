"""CPU-side checks of the C-ABI library (-m "not gpu"): it loads, exports every
entry point include/aakm.h declares, and validates arguments before any work
(no compute call needs a GPU).  Also the host-side sharding arithmetic."""
import ctypes as ct
import os
import subprocess

import pytest

from paper_1805_10638_b200 import aakm, synthetic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    if not os.path.exists(aakm.LIB_PATH):
        from paper_1805_10638_b200 import build
        build.build()
    return aakm.lib()


def test_exports_every_header_symbol(L):
    syms = aakm.header_symbols()
    assert len(syms) >= 19
    out = subprocess.run(["nm", "-D", "--defined-only", aakm.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        assert hasattr(L, s)


def test_library_is_sm100a_cuda(L):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", aakm.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_links_wheel_nccl_only(L):
    out = subprocess.run(["ldd", aakm.LIB_PATH], capture_output=True, text=True).stdout
    nccl = [ln for ln in out.splitlines() if "nccl" in ln]
    assert len(nccl) == 1 and "site-packages/nvidia/nccl" in nccl[0]


def test_abi_version_and_defaults(L):
    assert L.kmeans_abi_version() == 4
    c = aakm.Config()
    c.bounded = 7
    c.x_refresh = 3
    c.comm_always = 5
    c.fused_comm = 6
    assert L.kmeans_config_default(ct.byref(c)) == 0
    # PAPER.md:177 defaults; dense assignment unless asked for the bounded engine
    assert (c.m0, c.m_max, c.eps1, c.eps2, c.dynamic_m) == (2, 30, 0.02, 0.5, 1)
    assert c.bounded == 0 and c.x_refresh == 0 and c.comm_always == 0 and c.fused_comm == 0
    assert ct.sizeof(aakm.Config) == 64
    assert L.kmeans_config_default(None) == 1


def test_workspace_size_and_validation(L):
    c = aakm.config()
    n = ct.c_size_t()
    assert L.kmeans_workspace_size(1000, 16, 64, ct.byref(c), ct.byref(n)) == 0
    assert n.value > 1000 * 4 * 2
    n2 = ct.c_size_t()
    assert L.kmeans_workspace_size(2000, 16, 64, ct.byref(c), ct.byref(n2)) == 0 and n2.value > n.value
    for args in [(1000, 0, 64), (1000, 16, 0), (1000, 5000, 4)]:
        assert L.kmeans_workspace_size(*args, ct.byref(c), ct.byref(n)) == 1
    bad = aakm.config(m0=31)
    assert L.kmeans_workspace_size(1000, 16, 64, ct.byref(bad), ct.byref(n)) == 1
    bad = aakm.config(m_max=31, m0=2)
    assert L.kmeans_workspace_size(1000, 16, 64, ct.byref(bad), ct.byref(n)) == 1
    bad = aakm.config(eps1=0.6, eps2=0.5)
    assert L.kmeans_workspace_size(1000, 16, 64, ct.byref(bad), ct.byref(n)) == 1
    assert b"eps1" in L.kmeans_last_error(None)


def test_create_rejects_invalid_before_work(L):
    c = aakm.config()
    h = ct.c_void_p()
    # NULL X / workspace, k > n_global, uid mismatch -> INVALID without touching the device
    assert L.kmeans_create(ct.byref(h), None, 10, 10, 2, 3, ct.byref(c), None, 0, 0, 1, None, None) == 1
    assert L.kmeans_create(ct.byref(h), ct.c_void_p(256), 10, 10, 2, 11, ct.byref(c), ct.c_void_p(256),
                           1 << 30, 0, 1, None, None) == 1
    assert L.kmeans_create(ct.byref(h), ct.c_void_p(256), 10, 10, 2, 3, ct.byref(c), ct.c_void_p(256),
                           1 << 30, 0, 2, None, None) == 1
    assert L.kmeans_create(ct.byref(h), ct.c_void_p(256), 10, 10, 2, 3, ct.byref(c), ct.c_void_p(256),
                           16, 0, 1, None, None) == 1          # workspace too small
    assert b"workspace" in L.kmeans_last_error(None)


@pytest.mark.parametrize("N,world", [(10, 3), (16_000_000, 8), (7, 8), (100_000, 2)])
def test_shard_bounds_partition(N, world):
    spans = [synthetic.shard_bounds(N, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == N
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1
