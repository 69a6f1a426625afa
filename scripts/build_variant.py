"""Build a variant of libhbmc_b200.so with extra nvcc defines (A/B experiments).

    python scripts/build_variant.py TAG -DNAME=VAL ...   -> scratch_libs/libhbmc_TAG.so
Run a command against it on the GPU box with
    scripts/with_variant.sh TAG <command...>
which swaps it in for paper_1908_00741_b200/libhbmc_b200.so for the command
and restores the default build afterwards (the product itself always loads
its in-tree library).
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
from paper_1908_00741_b200 import _build as B  # noqa: E402

tag, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(REPO, "scratch_libs")
os.makedirs(out, exist_ok=True)
objs = []
for src, d, name in B.SOURCES:
    obj = os.path.join(B.OBJDIR, name + ".o")
    if src == "device.cu":
        obj = os.path.join(out, f"device_{tag}.o")
        cmd = [B.nvcc_path(), "-O3", "-std=c++17", *B.ARCH, "-lineinfo", "-Xptxas", "-O3",
               "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off,-O3", *defs, "-c", "-o", obj,
               os.path.join(B.CSRC, src)]
        subprocess.run(cmd, check=True)
    objs.append(obj)
lib = os.path.join(out, f"libhbmc_{tag}.so")
subprocess.run([B.nvcc_path(), *B.ARCH, "-shared", "-o", lib, *objs, "-lgomp"], check=True)
print(lib)
