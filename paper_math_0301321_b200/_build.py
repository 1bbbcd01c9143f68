"""Build libib_b200.so (the C-ABI of include/ib.h) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libib_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "ib.h")]


def nvcc() -> str:
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if p and os.path.exists(p):
            return p
    return "nvcc"


def build(force: bool = False, verbose: bool = False, extra=None, out: str = None) -> str:
    """nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo: each .cu compiled to an
    object in parallel (build/obj*/), then linked into the shared library."""
    target = out or SO
    newest = max(os.path.getmtime(p) for p in _deps())
    if not force and os.path.exists(target) and os.path.getmtime(target) >= newest:
        return target
    from concurrent.futures import ThreadPoolExecutor
    tag = f"{os.getpid()}"
    odir = os.path.join(HERE, "build", f"obj{tag}")
    os.makedirs(odir, exist_ok=True)
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
             "-I", os.path.join(ROOT, "include")]
    if verbose:
        flags.insert(0, "-Xptxas=-v")
    if extra:
        flags[0:0] = list(extra)
    objs = []

    def one(src):
        o = os.path.join(odir, os.path.basename(src) + ".o")
        subprocess.check_call([nvcc(), *flags, "-c", "-o", o, src])
        return o

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(one, sources()))
    tmp = target + f".tmp{tag}"
    subprocess.check_call([nvcc(), *ARCH, "-shared", "-cudart", "shared", "-o", tmp, *objs])
    os.replace(tmp, target)
    for o in objs:
        os.remove(o)
    os.rmdir(odir)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
