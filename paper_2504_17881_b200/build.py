"""Builds libps.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo
snapshot to the GPU box).  Usage: python -m paper_2504_17881_b200.build [--force]"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libps.so")
SRCS = [os.path.join(HERE, "csrc", f) for f in ("kernels.cu", "api.cpp", "planner.cpp")]
HDRS = [os.path.join(HERE, "csrc", "ps_internal.h"), os.path.join(ROOT, "include", "ps.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import nvidia.nccl  # the wheel torch itself loads
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc():
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if os.path.exists(cand) else "nvcc"


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    lib = out or LIB
    newest = max(os.path.getmtime(p) for p in SRCS + HDRS)
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= newest:
        return lib
    inc, libdir = nccl_dirs()
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-O2", "-shared",
           "-Xptxas", "-v" if verbose else "-O3",
           *[f"-D{d}" for d in defines],
           "-I", os.path.join(ROOT, "include"), "-I", inc, *SRCS, "-o", tmp,
           "-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{libdir}"]
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs, out=outs[0] if outs else None))
