"""Build libpga.so (sm_100a) in-tree with nvcc.

Usage: python -m paper_1403_4099_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpga.so")
CHECK_LIB = os.path.join(HERE, "libpga_check.so")   # -DPGA_DEVICE_CHECKS (tests only)
SOURCES = ["api.cu", "fitness.cu", "ga.cu", "corr.cu", "batch.cu", "stream.cu"]
HEADERS = ["pga_internal.cuh", os.path.join("..", "..", "include", "pga.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-warn-spills",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def _stale_lib(path) -> bool:
    if not os.path.exists(path):
        return True
    t = os.path.getmtime(path)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build_check(force: bool = False, verbose: bool = False) -> str:
    """The device-check variant (test infrastructure, tests/test_gpu_checks.py)."""
    if force or _stale_lib(CHECK_LIB):
        build(force=True, verbose=verbose, out=CHECK_LIB, defines=("PGA_DEVICE_CHECKS",))
    return CHECK_LIB


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    target = out or LIB
    if out is None and not force and not _stale():
        return LIB
    tmp = target + ".tmp%d" % os.getpid()
    cmd = [NVCC] + FLAGS + ["-D" + d for d in defines] + ["-o", tmp] + \
        [os.path.join(CSRC, s) for s in SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    args = sys.argv[1:]
    out = None
    defs = [a[2:] for a in args if a.startswith("-D")]
    if "-o" in args:
        out = args[args.index("-o") + 1]
    print(build(force="--force" in args, verbose=True, out=out, defines=defs))
