"""Build libsem.so in-tree for sm_100a with nvcc (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libsem.so")
SOURCES = ["kernels.cu", "sem_abi.cu", "matching.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _newest_input():
    paths = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(os.path.dirname(HERE), "include", "sem.h"), os.path.abspath(__file__)]
    return max(os.path.getmtime(p) for p in paths if os.path.isfile(p))


VARIANTS = {"": [], "_debug": ["-DSEM_DEBUG_CHECKS"]}   # libsem.so, libsem_debug.so (device bounds checks)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libsem.so (the product) and libsem_debug.so (the same sources with device-side bounds
    checks, SEM_DEBUG_CHECKS; used by tests/test_debug_checks_gpu.py) -- all nvcc runs in parallel."""
    os.makedirs(LIBDIR, exist_ok=True)
    libs = {v: os.path.join(LIBDIR, f"libsem{v}.so") for v in VARIANTS}
    newest = _newest_input()
    if not force and all(os.path.exists(l) and os.path.getmtime(l) >= newest for l in libs.values()):
        return LIB
    jobs = []
    for v, extra in VARIANTS.items():
        for src in SOURCES:
            obj = os.path.join(LIBDIR, src.replace(".cu", f"{v}.o"))
            cmd = [NVCC, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
            jobs.append((v, src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    objs = {v: [] for v in VARIANTS}
    for v, src, obj, proc in jobs:
        out, err = proc.communicate()
        if proc.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src} ({v or 'release'}):\n{out}\n{err}")
        if verbose and not v:
            sys.stderr.write(err)
        objs[v].append(obj)
    for v, lib in libs.items():
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs[v], "-o", lib + ".tmp",
               "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(lib + ".tmp", lib)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
