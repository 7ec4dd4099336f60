"""Build libeat.so (the C-ABI library) in-tree for sm_100a with nvcc.

Sources: paper_1912_00966_b200/csrc/{build.cpp, kernels.cu, partition.cu,
api.cu}; public header include/eat.h.  NCCL is the torch-bundled one
(nvidia/nccl in site-packages), linked with an rpath so the same libnccl is
used by torch.distributed and by libeat in one process.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "eat")
LIB = os.path.join(PKG, "libeat.so")
SOURCES = ["build.cpp", "kernels.cu", "partition.cu", "async.cu", "peer.cu", "cluster.cu", "gasync.cu", "api.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations or []) if spec else []:
        inc, lib = os.path.join(base, "nccl", "include"), os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("nccl.h not found under site-packages/nvidia/nccl")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    inc, libdir = nccl_dirs()
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "eat.h"))
    objs = []
    procs = []
    for src in SOURCES:  # translation units compile in parallel
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if not force and not _stale(obj, [path] + headers):
            continue
        cmd = [nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-O3,-pthread",
               "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc, "-c", path, "-o", obj]
        if src.endswith(".cpp"):
            cmd[1:1] = ["-x", "cu"]
        if ptxas_v:
            cmd += ["-Xptxas", "-v"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd), cmd, obj))
    failed = None
    for p, cmd, obj in procs:
        if p.wait() != 0:
            failed = failed or subprocess.CalledProcessError(p.returncode, cmd)
            if os.path.exists(obj):
                os.remove(obj)  # never link a stale object
    if failed:
        raise failed
    if force or _stale(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [nvcc(), "-shared", *ARCH, "-o", tmp, *objs, "-L", libdir, "-l:libnccl.so.2",
               "-Xlinker", "-rpath," + libdir, "-lpthread"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_v="-v" in sys.argv)
