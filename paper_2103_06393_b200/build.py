"""Build libtuckmat_b200.so in-tree (nvcc for sm_100a, g++ for host C++).

The shared library is the product: the C ABI of include/tuckmat_b200.h, the
CUDA kernels and the C++ drop-in of include/tuckmat_b200/tuckmat.hpp.  It is
built in the package directory so it travels to the GPU box with the repo.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libtuckmat_b200.so")
BUILD = os.path.join(ROOT, "build", "tuckmat_b200")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU_SOURCES = ["tm_capi.cu"]
CPP_SOURCES = ["tm_io.cpp", "tm_dropin.cpp"]
HEADERS_DIRS = [CSRC, os.path.join(ROOT, "include")]


def _sources_mtime():
    m = 0.0
    for d in HEADERS_DIRS:
        for dp, _, fs in os.walk(d):
            for f in fs:
                if f.endswith((".cu", ".cuh", ".cpp", ".h", ".hpp")):
                    m = max(m, os.path.getmtime(os.path.join(dp, f)))
    return max(m, os.path.getmtime(__file__))


def needs_build():
    return not os.path.exists(OUT) or os.path.getmtime(OUT) < _sources_mtime()


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(force=False, verbose=False, ptxas_verbose=False):
    if not force and not needs_build():
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    for src in CU_SOURCES:
        obj = os.path.join(BUILD, src + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler",
               "-fPIC,-fvisibility=hidden", *inc, "-c", os.path.join(CSRC, src), "-o", obj]
        if ptxas_verbose:
            cmd.insert(1, "-Xptxas=-v")
        # diagnostics builds, e.g. TMB_NVCC_FLAGS=-DTMB_TC_PROFILE (forward wait profile)
        cmd[1:1] = os.environ.get("TMB_NVCC_FLAGS", "").split()
        _run(cmd, verbose)
        objs.append(obj)
    for src in CPP_SOURCES:
        obj = os.path.join(BUILD, src + ".o")
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-fvisibility=hidden", *inc, "-I",
               os.path.join(CUDA_HOME, "include"), "-c", os.path.join(CSRC, src), "-o", obj]
        _run(cmd, verbose)
        objs.append(obj)
    tmp = OUT + ".tmp"
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-ldl", "-lpthread"], verbose)
    shutil.move(tmp, OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_verbose="--ptxas" in sys.argv)
    print(OUT)
