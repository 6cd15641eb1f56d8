"""Build libmrf.so (the C-ABI library of include/mrf.h) with nvcc for sm_100a, in tree."""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libmrf.so")
# the checked build (MRF_CHECK=1: device-side bounds checks on the hot kernels' data-dependent
# indices; SURVEY §4 T8 while compute-sanitizer is unavailable on the GPU pool)
LIB_CHECKED = os.path.join(HERE, "libmrf_checked.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl"))
    cands.append(os.path.join(sys.prefix, "lib", f"python{sys.version_info.major}.{sys.version_info.minor}",
                              "site-packages", "nvidia", "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    raise RuntimeError("nccl.h not found (expected the torch-bundled nvidia/nccl package)")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu"))) + sorted(glob.glob(os.path.join(CSRC, "*.cuh")))


def needs_build(lib=None) -> bool:
    lib = lib or LIB
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = sources() + [os.path.join(INCLUDE, "mrf.h"), os.path.abspath(__file__)]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, extra=(), out=None) -> str:
    out = out or LIB
    if not force and not needs_build(out):
        return out
    inc, libdir = nccl_dirs()
    cus = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    tmp = out + f".tmp{os.getpid()}"
    cmd = [NVCC, "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-O2", "-shared",
           "-Xptxas", "-v" if verbose else "-O3",
           "-I", INCLUDE, "-I", inc, *cus, "-o", tmp,
           "-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{libdir}", *extra]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    if verbose:
        print(r.stdout + r.stderr)
    os.replace(tmp, out)
    return out


def build_checked(force: bool = False) -> str:
    return build(force=force, extra=("-DMRF_CHECK=1",), out=LIB_CHECKED)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
    if "--checked" in sys.argv:
        print(build_checked(force="--force" in sys.argv))
