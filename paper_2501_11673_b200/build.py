"""Build libkpp.so (the C-ABI library) in-tree with nvcc for sm_100a.

Product build helper: compiles paper_2501_11673_b200/csrc/*.cu against include/kpp.h
and the NCCL that torch ships (the same libnccl.so.2 the process already loads).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# A/B experiments: KPP_LIB names another library file, KPP_NVCC_FLAGS adds compiler flags (objects go
# to a directory of their own); the product build uses neither
LIB = os.environ.get("KPP_LIB") or os.path.join(HERE, "libkpp.so")
EXTRA = os.environ.get("KPP_NVCC_FLAGS", "").split()
OBJDIR = os.path.join(HERE, "build" if not os.environ.get("KPP_LIB") else "build_" + os.path.basename(LIB).replace(".so", ""))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    try:
        import nvidia.nccl as nn  # torch's NCCL wheel
        base = list(nn.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(ROOT, "include", "*.h")))


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in sources() + headers() + [__file__])


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    # one builder at a time (torchrun starts one process per GPU): the others wait on the lock and
    # then find the library up to date; the library is linked to a temporary name and renamed, so a
    # concurrent loader never sees a partial file
    import fcntl
    os.makedirs(OBJDIR, exist_ok=True)
    with open(os.path.join(OBJDIR, ".lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if not force and up_to_date():
            return LIB
        return _build_locked(verbose)


def _build_locked(verbose: bool) -> str:
    inc, lib = nccl_dirs()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    objdir = OBJDIR
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc, *ARCH, *EXTRA, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xptxas", "-v" if verbose else "-O3", "-I", inc, "-I", os.path.join(ROOT, "include"),
               "-c", src, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out.decode())
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed")
    tmp = LIB + ".tmp"
    cmd = [nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-L", lib, "-l:libnccl.so.2",
           "-Xlinker", f"-rpath={lib}", "-lcudart"]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
