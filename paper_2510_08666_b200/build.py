"""Build libdinfer.so (all CUDA kernels + the C ABI) in-tree for sm_100a.

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, linked against the
NCCL that torch loads (nvidia-nccl wheel, 2.28.x) with an rpath to it, so the
library and torch share one libnccl.so.2.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libdinfer.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations or []) if spec else []:
        inc, lib = os.path.join(base, "nccl", "include"), os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    return None, None


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + glob.glob(os.path.join(PKG, "csrc", "*.h"))
    deps.append(os.path.join(ROOT, "include", "dinfer.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    inc, lib = nccl_paths()
    cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-shared",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(PKG, "csrc")]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    if inc:
        cmd += ["-DDINFER_WITH_NCCL", "-I", inc]
    cmd += os.environ.get("DINFER_EXTRA_NVCC", "").split()  # diagnostics, e.g. -DDINFER_DEBUG_HANG
    cmd += sources()
    tmp = LIB + ".tmp"
    cmd += ["-o", tmp]
    if lib:
        cmd += ["-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libdinfer.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
