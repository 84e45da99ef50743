"""Build ``libams_b200.so`` (sm_100a) in-tree with nvcc.

    python -m paper_1410_6754_b200.build [--force]

The library is the C ABI of include/ams_b200.h; it is loaded with ctypes by
``paper_1410_6754_b200._lib``.  Every source is compiled to an object under
``lib/obj`` (in parallel, only when it or a header changed) and the objects
are linked into the shared library.  Built artefacts stay in-tree
(git-ignored) so they travel to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "lib")
OBJ_DIR = os.path.join(LIB_DIR, "obj")
LIB = os.path.join(LIB_DIR, "libams_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) +
                  glob.glob(os.path.join(CSRC, "host", "*.cpp")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) +
                  glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(ROOT, "include", "*.h")))


def obj_of(src: str) -> str:
    return os.path.join(OBJ_DIR, os.path.basename(src) + ".o")


def stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(p) > t for p in deps)


def up_to_date() -> bool:
    return not stale(LIB, sources() + headers())


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(OBJ_DIR, exist_ok=True)
    hdrs = headers()
    todo = [s for s in sources() if force or stale(obj_of(s), [s] + hdrs)]
    inc = ["-I", os.path.join(ROOT, "include")]
    with ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as pool:
        list(pool.map(lambda s: _run([NVCC, *ARCH, *FLAGS, *inc, "-c", s, "-o", obj_of(s)], verbose), todo))
    tmp = LIB + ".tmp"
    _run([NVCC, *ARCH, "-shared", *[obj_of(s) for s in sources()], "-o", tmp], verbose)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
