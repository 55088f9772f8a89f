"""Build recipe for libppfg.so (sm_100a only), in-tree so the .so travels with
the repo snapshot to the GPU box."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
SO = os.path.join(PKG, "libppfg.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off",
]
OBJ_DIR = os.path.join(PKG, "_obj")


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


# host-only C++ units (compiled by nvcc as plain C++, per-unit ISA flags)
HOST_FLAGS = {"hostcopy.cpp": ["-Xcompiler", "-mavx2"]}


def units():
    """The translation units: ppfg.cu (host code + small kernels), the
    tab_*.cu kernel-table units and the host-only *.cpp units, compiled in
    parallel."""
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def compile_cmd(src, obj):
    """nvcc command compiling one unit (a .cpp unit is host C++ only)."""
    extra = HOST_FLAGS.get(os.path.basename(src), [])
    return [_nvcc(), *NVCC_FLAGS, *extra, "-I" + INCLUDE, "-c", "-o", obj, src]


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
                  + glob.glob(os.path.join(INCLUDE, "*.h")))


def sources():
    return units() + headers()


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(s) > t for s in sources())


def _obj(cu):
    return os.path.join(OBJ_DIR, os.path.splitext(os.path.basename(cu))[0] + ".o")


def build(force: bool = False, verbose: bool = False, jobs: int = 0) -> str:
    if not force and not stale():
        return SO
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(OBJ_DIR, exist_ok=True)
    newest_header = max(os.path.getmtime(h) for h in headers())

    def compile_one(cu):
        obj = _obj(cu)
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(
                os.path.getmtime(cu), newest_header):
            return obj
        tmp = obj + f".tmp{os.getpid()}"
        cmd = compile_cmd(cu, tmp)
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        os.replace(tmp, obj)
        return obj

    jobs = jobs or min(len(units()), os.cpu_count() or 1)
    with ThreadPoolExecutor(max_workers=jobs) as ex:
        objs = list(ex.map(compile_one, units()))
    tmp = SO + f".tmp{os.getpid()}"
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(SO)
