"""Build the libraries in-tree for sm_100a (nvcc -shared -Xcompiler -fPIC).

    libpe.so       the product: include/pe.h (pe.cu, bm.cu)
    libpe_test.so  modular-core probes and roofline microbenchmarks: include/pe_test.h (probe.cu);
                   loaded only by tests/, bench.py and scripts/

    python -m paper_2004_11571_b200.build [--force]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libpe.so")
TEST_LIB = os.path.join(PKG, "libpe_test.so")
LIBS = {LIB: [os.path.join(CSRC, "pe.cu"), os.path.join(CSRC, "bm.cu"), os.path.join(CSRC, "fast.cu")],
        TEST_LIB: [os.path.join(CSRC, "probe.cu")]}
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _stale(lib) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = (glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
            + glob.glob(os.path.join(ROOT, "include", "*.h")) + [__file__])
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    for lib, sources in LIBS.items():
        if force or _stale(lib):
            _build_one(lib, sources, verbose)
    return LIB


def _build_one(LIB, SOURCES, verbose):
    objs = []
    logs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, os.path.basename(src) + f".{os.getpid()}.o")
        r = subprocess.run([NVCC, *FLAGS, "-c", src, "-o", obj], capture_output=True, text=True)
        logs.append(r.stdout + r.stderr)
        if r.returncode != 0:
            for o in objs:
                os.unlink(o)
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        objs.append(obj)
    tmp = LIB + f".tmp{os.getpid()}"
    r = subprocess.run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs],
                       capture_output=True, text=True)
    for o in objs:
        os.unlink(o)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(os.path.join(CSRC, os.path.basename(LIB) + ".ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
