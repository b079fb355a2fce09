"""Build libmvgs.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

The library is rebuilt when a source is newer than it OR when the compile flags differ from
the ones it was built with (stamped next to it), so a library built with experiment knobs
(MVGS_NVCC_EXTRA, e.g. -DMVGS_NO_CULL) is never silently reused by build() / smoke().
Experiments build into their own path with MVGS_LIB=/path/to/variant.so (the binding loads
the same variable), leaving the product library untouched.
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("MVGS_LIB", os.path.join(HERE, "libmvgs.so"))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(HERE, "..", "include", "mvgs.h")]


def _flags(extra):
    return " ".join(FLAGS + extra)


def _stamp_path(lib):
    return lib + ".flags"


def build(force: bool = False, verbose: bool = False, lib: str | None = None) -> str:
    lib = lib or LIB
    extra = os.environ.get("MVGS_NVCC_EXTRA", "").split()  # experiments, e.g. -DMVGS_RS_IPT=12
    want = hashlib.sha256(_flags(extra).encode()).hexdigest()
    have = open(_stamp_path(lib)).read().strip() if os.path.exists(_stamp_path(lib)) else ""
    newest = max(os.path.getmtime(p) for p in deps())
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= newest and have == want:
        return lib
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, *extra, *(["-Xptxas", "-v"] if verbose else []), *sources(), "-o", tmp]
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    with open(_stamp_path(lib), "w") as f:
        f.write(want + "\n")
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=True))
