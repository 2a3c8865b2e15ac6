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
SOURCES = ["sem_kernels.cu", "ax_tma.cu", "ax_tma_mass.cu", "ax_tma_pc.cu", "cg_update.cu", "sem_host.cpp",
           "sem_comm.cu", "fd2d.cu", "ax_tma_sr.cu", "cg_sr.cu", "cg_resident.cu"]
HEADERS = ["sem_internal.h", "sem_comm.h", "p2p_dev.cuh", "cg_device.cuh", "ax_tma.cuh", "ax_dmma.cuh", "ax_dmmag.cuh"]
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
    deps.append(os.path.join(ROOT, "include", "fd.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = True) -> str:
    """Compile the translation units in parallel (nvcc -c; objects cached under
    build/ and recompiled when their source or any header is newer), then link."""
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    inc, lib = nccl_dirs()
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    common = ["nvcc", *ARCH, *os.environ.get("SEM_NVCC_EXTRA", "").split(), "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-O2", "-Xptxas", "-warn-spills",
              "-I", os.path.join(ROOT, "include"), "-I", inc]
    hdr = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "sem.h"),
                                                     os.path.join(ROOT, "include", "fd.h"),
                                                     os.path.abspath(__file__)]
    newest_hdr = max(os.path.getmtime(h) for h in hdr)
    objs = [os.path.join(objdir, os.path.splitext(f)[0] + ".o") for f in SOURCES]

    def stale(f, o):
        if force or not os.path.exists(o):
            return True
        t = os.path.getmtime(o)
        return os.path.getmtime(os.path.join(CSRC, f)) > t or newest_hdr > t

    cmds = [common + ["-c", os.path.join(CSRC, f), "-o", o]
            for f, o in zip(SOURCES, objs) if stale(f, o)]
    if verbose and cmds:
        print(" ".join(cmds[0]), "... (x%d, parallel)" % len(cmds), file=sys.stderr)
    with ThreadPoolExecutor(max_workers=max(1, len(cmds))) as ex:
        procs = list(ex.map(lambda c: subprocess.run(c, cwd=CSRC, capture_output=True, text=True),
                            cmds))
    for c, p in zip(cmds, procs):
        if verbose and p.stderr:
            sys.stderr.write(p.stderr)
        if p.returncode != 0:
            if os.path.exists(c[-1]):
                os.remove(c[-1])
            raise subprocess.CalledProcessError(p.returncode, c, p.stdout, p.stderr)
    tmp = LIB + ".tmp"
    link = ["nvcc", *ARCH, "--shared", *objs, "-o", tmp, "-L", lib, "-l:libnccl.so.2",
            "-Xlinker", f"-rpath={lib}", "-lcudart"]
    subprocess.check_call(link, cwd=CSRC)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
