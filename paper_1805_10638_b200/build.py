"""Build libaakm.so in-tree: nvcc for sm_100a (-gencode arch=compute_100a,code=sm_100a),
linked against the torch-wheel NCCL (the same libnccl.so.2 torch loads)."""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libaakm.so")
BUILD = os.path.join(HERE, "_build")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir():
    for p in sys.path + [sysconfig.get_paths()["purelib"]]:
        cand = os.path.join(p, "nvidia", "nccl")
        if os.path.exists(os.path.join(cand, "include", "nccl.h")):
            return cand
    raise RuntimeError("torch-wheel NCCL (nvidia/nccl) not found")


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    global OUT, BUILD
    if out:                                  # A/B variant builds (tools/): another .so and build dir
        OUT, BUILD = out, out + ".build"
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "aakm.h")]
    nd = nccl_dir()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    flags = ["-O3", "-std=c++17", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
             "-I", os.path.join(nd, "include"), "-I", os.path.join(ROOT, "include"),
             "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills",
             *os.environ.get("AAKM_NVCC_EXTRA", "").split()]     # perf experiments only (A/B variants)
    # content stamp (sources + flags): mtimes alone missed edits made while a build ran
    h = hashlib.sha256(" ".join(flags).encode())
    for p in srcs + hdrs:
        h.update(p.encode())
        with open(p, "rb") as f:
            h.update(f.read())
    stamp = os.path.join(BUILD, "stamp")
    digest = h.hexdigest()
    if not force and os.path.exists(OUT) and os.path.exists(stamp) and open(stamp).read() == digest:
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    procs = []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s) + ".o")
        objs.append(o)
        cmd = [nvcc, *flags, "-DAAKM_BUILD", "-c", s, "-o", o]
        if verbose:
            print(" ".join(cmd))
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd) + "\n" + out.decode())
        if verbose and out:
            print(out.decode())
    tmp = OUT + f".{os.getpid()}.tmp"
    lib = os.path.join(nd, "lib")
    cmd = [nvcc, "-shared", *ARCH, "-o", tmp, *objs, "-L", lib, "-l:libnccl.so.2",
           "-Xlinker", "-rpath=" + lib]
    subprocess.check_call(cmd)
    os.replace(tmp, OUT)
    with open(stamp, "w") as f:
        f.write(digest)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
