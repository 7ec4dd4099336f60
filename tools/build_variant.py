"""Build an experimental libeat.so variant with extra -D defines into ab/
(for same-box A/B with tools/ab_lib.py).  Usage:
  python tools/build_variant.py NAME [-DFOO ...]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_00966_b200 import build_ext as B

name, defs = sys.argv[1], sys.argv[2:]
bdir = os.path.join(B.ROOT, "build", "var_" + name)
os.makedirs(bdir, exist_ok=True)
os.makedirs(os.path.join(B.ROOT, "ab"), exist_ok=True)
inc, libdir = B.nccl_dirs()
objs = []
procs = []
for src in B.SOURCES:
    obj = os.path.join(bdir, src + ".o")
    objs.append(obj)
    cmd = [B.nvcc(), "-O3", "-std=c++17", *B.ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-O3,-pthread", *defs,
           "-I", os.path.join(B.ROOT, "include"), "-I", B.CSRC, "-I", inc, "-c", os.path.join(B.CSRC, src), "-o", obj]
    if src.endswith(".cpp"):
        cmd[1:1] = ["-x", "cu"]
    procs.append(subprocess.Popen(cmd, stderr=subprocess.DEVNULL if "-q" in os.environ.get("BV", "") else None))
for p in procs:
    assert p.wait() == 0
out = os.path.join(B.ROOT, "ab", f"libeat_{name}.so")
subprocess.check_call([B.nvcc(), "-shared", *B.ARCH, "-o", out, *objs, "-L", libdir, "-l:libnccl.so.2",
                       "-Xlinker", "-rpath," + libdir, "-lpthread"])
print(out)
