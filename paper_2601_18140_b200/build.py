"""Build the product library in-tree: paper_2601_18140_b200/lib/librtlsim.so.

nvcc cross-compiles sm_100a without a GPU.  Flags: -gencode
arch=compute_100a,code=sm_100a -lineinfo -O3.  The CUDA runtime is linked
statically (one .so to ship to the GPU box).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "librtlsim.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["runtime.cu", "compiler.cpp", "passes.cpp", "codegen.cpp"]
HEADERS = ["kernels.cuh", "lanes.cuh", "lanes_t.cuh", "gather_brx.cuh", "lanes_b.cuh", "gather_b.cuh", "lanes_r.cuh", "single.cuh", "repcut.cuh", "compiler.hpp", "codegen.hpp"]


def _newest_input() -> float:
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "rtlsim.h"))
    files.append(os.path.abspath(__file__))
    return max(os.path.getmtime(f) for f in files)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    lib = out or LIB
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= _newest_input():
        return lib
    cmd = [NVCC, "-std=c++17", "-O3", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-O3", "-shared",
           "-I", os.path.join(ROOT, "include"),
           *["-D" + d for d in defines],
           *[os.path.join(CSRC, f) for f in SOURCES], "-ldl", "-o", lib + ".tmp"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv or bool(defs), verbose="-v" in sys.argv,
                out=outs[0] if outs else None, defines=defs))
