"""In-tree build of the CUDA extension (libacz_gpu.so) for sm_100a.

The shared library is the C-ABI declared in include/acz_gpu.h. It is built with plain
nvcc (no torch JIT cache) so the .so lives in-tree and travels to the GPU box.
Every kernel translation unit is compiled with --fmad=false (no FMA contraction, the
reference's arithmetic order: SURVEY.md sec. 0 fact 4) and -lineinfo for ncu source pages.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libacz_gpu.so")
SOURCES = ["stats.cu", "quant.cu", "quant_spec.cu", "huffman.cu", "decode.cu", "api.cu"]
HEADERS = ["common.cuh", "internal.h"]

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
EXTRA = os.environ.get("ACZ_NVCC_EXTRA", "").split()
FLAGS = EXTRA + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
         "-Xptxas", "-warn-spills", f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "acz_gpu.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(LIBDIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd))
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose and out:
            sys.stdout.write(out.decode())
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


CPP_TEST_SRC = os.path.join(ROOT, "tests", "cpp", "test_host.cpp")
CPP_TEST_BIN = os.path.join(ROOT, "tests", "cpp", "test_host")


def build_cpp_test(force: bool = False) -> str:
    """Builds the C++ host-layer test (cpp/acz_b200.hpp over libacz_gpu.so) with g++."""
    hdr = os.path.join(HERE, "cpp", "acz_b200.hpp")
    if (not force and os.path.exists(CPP_TEST_BIN)
            and all(os.path.getmtime(CPP_TEST_BIN) > os.path.getmtime(d)
                    for d in (CPP_TEST_SRC, hdr, LIB))):
        return CPP_TEST_BIN
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", f"-I{os.path.join(ROOT, 'include')}",
           f"-I{os.path.join(HERE, 'cpp')}", CPP_TEST_SRC, "-o", CPP_TEST_BIN, f"-L{LIBDIR}",
           "-lacz_gpu", "-Wl,-rpath,$ORIGIN/../../paper_2011_09017_b200/lib"]
    subprocess.run(cmd, check=True)
    return CPP_TEST_BIN


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
