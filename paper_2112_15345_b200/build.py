"""Build the in-tree sm_100a shared library ``libegonet.so`` with nvcc.

Every kernel is compiled to SASS for sm_100a (no PTX JIT on the box); the .so is
built in-tree so that it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(PKG, "libegonet.so")
HEADERS = [os.path.join(ROOT, "include", "egonet.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-I", os.path.join(ROOT, "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale(so: str = SO) -> bool:
    if not os.path.exists(so):
        return True
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + HEADERS
    return os.path.getmtime(so) < max(os.path.getmtime(d) for d in deps)


SO_CHECK = os.path.join(PKG, "libegonet_check.so")


def build(force: bool = False, verbose: bool = False, check: bool = False) -> str:
    """check: the bounds-checked variant libegonet_check.so (-DEG_CHECK=1: device-side
    asserts on the hot paths' indices; load it with EG_LIB=<path>)."""
    so = SO_CHECK if check else SO
    if not force and not _stale(so):
        return so
    tmp = so + f".tmp{os.getpid()}"
    cmd = ["nvcc", *NVCC_FLAGS, *(["-DEG_CHECK=1"] if check else []), "-shared", "-o", tmp, *sources()]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, so)
    return so


def build_variant(name: str, defines) -> str:
    """A/B builds: libegonet_<name>.so with extra -D defines (load with EG_LIB=<path>)."""
    so = os.path.join(PKG, f"libegonet_{name}.so")
    tmp = so + f".tmp{os.getpid()}"
    cmd = ["nvcc", *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-shared", "-o", tmp, *sources()]
    subprocess.check_call(cmd)
    os.replace(tmp, so)
    return so


if __name__ == "__main__":
    if "--variant" in sys.argv:   # build.py --variant NAME DEF=VAL ...
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], sys.argv[i + 2:]))
        sys.exit(0)
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, check="--check" in sys.argv))
