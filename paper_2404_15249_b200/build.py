"""Build the in-tree CUDA library lib/libkfbi.so for sm_100a (nvcc; no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib", "libkfbi.so")
SOURCES = ["api.cu", "kernels2d.cu", "kernels3d.cu", "setup_gpu.cu", "setup2d.cpp", "setup3d.cpp"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC,-fopenmp,-O2"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "kfbi.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def nccl_paths():
    """Compile and link against the NCCL that torch loads (pip nvidia-nccl), rpath to it."""
    try:
        import nvidia.nccl as nn   # noqa: F401
        root = os.path.dirname(nn.__file__) if getattr(nn, "__file__", None) else list(nn.__path__)[0]
    except Exception:
        root = None
    if root and os.path.exists(os.path.join(root, "include", "nccl.h")):
        lib = os.path.join(root, "lib")
        return ["-I" + os.path.join(root, "include"), "-L" + lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib]
    return ["-lnccl"]


def build(force: bool = False, verbose: bool = False) -> str:
    """Each source compiles to an object in parallel (no relocatable device code), then one link."""
    if not force and not stale():
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    objdir = os.path.join(HERE, "lib", "obj")
    os.makedirs(objdir, exist_ok=True)
    inc = nccl_paths()
    inc = [a for a in inc if a.startswith("-I")]

    def compile_one(src):
        obj = os.path.join(objdir, src + ".o")
        extra = os.environ.get("KFBI_NVCC_EXTRA", "").split()   # e.g. -DKFBI_BOUNDS (device index checks)
        cmd = [nvcc()] + NVCC_FLAGS + extra + inc + ["-c", "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True, cwd=CSRC)
        return obj

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    cmd = ([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB + ".tmp"] + objs
           + ["-lgomp"] + nccl_paths())
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
