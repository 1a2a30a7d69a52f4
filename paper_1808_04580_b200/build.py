"""Builds the B200 extension in-tree: paper_1808_04580_b200/libfgs_b200.so.

nvcc -gencode arch=compute_100a,code=sm_100a (sm_100a only), -lineinfo so
ncu's source page maps to csrc/, objects compiled in parallel, linked against
cuFFT and NCCL from the CUDA toolkit / system.  Usage: python -m
paper_1808_04580_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# FGS_BUILD_TAG=x (tuning builds with FGS_NVCC_DEFINES): libfgs_b200_x.so
# from build/obj_x, loaded by tools/variant_bench.py; never the product path
_TAG = os.environ.get("FGS_BUILD_TAG", "")
OUT = os.path.join(HERE, f"libfgs_b200_{_TAG}.so" if _TAG else "libfgs_b200.so")
OBJ = os.path.join(ROOT, "build", f"obj_{_TAG}" if _TAG else "obj")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

SOURCES = ["core.cu", "lanczos.cu", "capi.cu", "peak.cu", "kmeans.cu", "cg.cu", "nystrom.cu", "workload.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++20", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), "-I", CSRC]
NVFLAGS = ARCH + ["-lineinfo", "--expt-relaxed-constexpr", "-Xptxas", "-O3"]
# tuning builds: extra nvcc defines, e.g. FGS_NVCC_DEFINES="FGS_INTERP12_MINB=3"
NVFLAGS += ["-D" + d for d in os.environ.get("FGS_NVCC_DEFINES", "").split() if d]


def _deps():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "fgs_b200.h")]
    return max(os.path.getmtime(f) for f in files)


def _compile(src: str, verbose: bool) -> str:
    os.makedirs(OBJ, exist_ok=True)
    obj = os.path.join(OBJ, os.path.splitext(src)[0] + ".o")
    path = os.path.join(CSRC, src)
    if src.endswith(".cu"):
        cmd = [NVCC] + COMMON + NVFLAGS + ["-c", path, "-o", obj]
    else:
        cmd = ["g++", "-O3", "-std=c++20", "-fPIC", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
               "-I", os.path.join(CUDA, "include"), "-c", path, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= _deps():
        if not _TAG:
            build_cli(verbose)
        return OUT
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    link = [NVCC] + ARCH + ["-shared", "-o", OUT] + objs + [
        "-L", os.path.join(CUDA, "lib64"), "-lcufft", "-lcusolver", "-lcublas", "-lcudart", "-ldl",
        "-Xlinker", "-rpath=" + os.path.join(CUDA, "lib64")]
    if verbose:
        print(" ".join(link), flush=True)
    subprocess.run(link, check=True)
    if not _TAG:
        build_cli(verbose)
    return OUT


CLI_SRC = os.path.join(HERE, "cli", "fgs_b200_cli.cpp")
CLI_OUT = os.path.join(HERE, "fgs-b200")


def build_cli(verbose: bool = False) -> str:
    """The command-line drivers (tools/commands.cpp analogue) linked against
    the in-tree library with an $ORIGIN rpath."""
    if (os.path.exists(CLI_OUT) and os.path.getmtime(CLI_OUT) >= os.path.getmtime(OUT)
            and os.path.getmtime(CLI_OUT) >= max(os.path.getmtime(CLI_SRC),
                                                 os.path.getmtime(os.path.join(ROOT, "include", "fgs", "b200.hpp")))):
        return CLI_OUT
    cmd = ["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"), CLI_SRC, "-L", HERE, "-lfgs_b200",
           "-Wl,-rpath,$ORIGIN", "-o", CLI_OUT]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return CLI_OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
