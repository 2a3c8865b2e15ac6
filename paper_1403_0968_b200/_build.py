"""Build libsem.so (sm_100a) in-tree with nvcc.  No torch types cross the ABI;
the .so is loaded by paper_1403_0968_b200/sem.py through ctypes."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libsem.so")
SOURCES = ["sem_kernels.cu", "ax_tma.cu", "cg_update.cu", "sem_host.cpp", "sem_comm.cu"]
HEADERS = ["sem_internal.h", "sem_comm.h", "cg_device.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return os.path.join(d, "include"), os.path.join(d, "lib")
    raise RuntimeError("NCCL headers (nvidia/nccl from the torch wheel) not found")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "sem.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and not needs_build():
        return LIB
    inc, lib = nccl_dirs()
    tmp = LIB + ".tmp"
    cmd = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-O2", "--shared", "-Xptxas", "-warn-spills",
           "-I", os.path.join(ROOT, "include"), "-I", inc,
           *[os.path.join(CSRC, f) for f in SOURCES],
           "-o", tmp, "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}",
           "-lcudart"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
