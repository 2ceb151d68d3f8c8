"""Build libcacsi.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_1603_06400_b200.build [--verbose]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcacsi.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-O3", "-std=c++17", "-lineinfo", "--ftz=true",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-I", os.path.join(ROOT, "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "cacsi.h"), os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


LIB_CHECKED = os.path.join(HERE, "libcacsi_checked.so")


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """checked=True: libcacsi_checked.so with the device-side bounds checks (CACSI_CHECK)."""
    lib = LIB_CHECKED if checked else LIB
    if not force and not checked and not _stale():
        return lib
    extra = ["-Xptxas", "-v"] if verbose else []
    if checked:
        extra += ["-DCACSI_CHECKS"]
    cmd = [NVCC, *FLAGS, *extra, "-shared", "-o", lib + ".tmp", *sources()]
    # exported symbols: only the extern "C" cacsi_* entry points
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose="--verbose" in sys.argv, checked="--checked" in sys.argv))
