"""In-tree build of libhbmc_b200.so (host builder + sm_100a kernels).

Each translation unit is compiled to an object in parallel (nvcc for .cu,
sm_100a only, -lineinfo; the C++ host builder with -ffp-contract=off), then
linked into one shared library next to this file, so the .so travels with
the repository snapshot to the GPU box.
"""

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhbmc_b200.so")
OBJDIR = os.path.join(CSRC, "build")
# (source, extra defines, object name)
SOURCES = [("builder.cpp", [], "builder"), ("device.cu", [], "device"),
           ("dist.cu", [], "dist"), ("ic0.cu", [], "ic0"),
           ("mm_parse.cpp", [], "mm_parse")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path():
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; cannot build libhbmc_b200.so")
    return cand


def _deps():
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)
            if f.endswith((".cu", ".cuh", ".cpp", ".h"))]
    deps.append(os.path.join(HERE, "..", "include", "hbmc_b200.h"))
    deps.append(os.path.abspath(__file__))
    return deps


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in _deps() if os.path.exists(d))


def _compile(spec, verbose):
    src, defs, name = spec
    obj = os.path.join(OBJDIR, name + ".o")
    cmd = [nvcc_path(), "-O3", "-std=c++17", *ARCH, "-lineinfo",
           "-Xptxas", "-v" if verbose else "-O3",
           "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off,-O3",
           *defs, "-c", "-o", obj, os.path.join(CSRC, src)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    return obj, res


def build(force=False, verbose=False):
    if not force and not needs_build():
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    failed = False
    for obj, res in results:
        if verbose or res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
        failed |= res.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed building libhbmc_b200.so")
    cmd = [nvcc_path(), *ARCH, "-shared", "-o", LIB + ".tmp",
           *[obj for obj, _ in results], "-lgomp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed for libhbmc_b200.so")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
