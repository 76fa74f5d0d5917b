"""Build libswe_b200.so in-tree: nvcc for the sm_100a device code, g++ for the
host builders (compiled with -ffp-contract=off, reading A19)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libswe_b200.so")
BUILD = os.path.join(HERE, "_build")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dirs():
    """NCCL headers/library: the copy torch loads (nvidia-nccl wheel), else the system one."""
    try:
        import nvidia.nccl as _n
        base = list(_n.__path__)[0]
        return os.path.join(base, "include"), os.path.join(base, "lib")
    except Exception:
        return "/usr/include", "/usr/lib/x86_64-linux-gnu"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
HOST_SRC = ["refel.cpp", "mesh.cpp"]
CU_SRC = ["solver.cu"]
DEPS = ["host.hpp", "kernels.cuh"]


def _stale(out: str, inputs: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(i) > t for i in inputs)


def build(force: bool = False, verbose: bool = False, defines: tuple = (), out: str | None = None) -> str:
    """defines/out: build an A/B variant (e.g. ("VOL_UNROLL=2",), "libswe_u2.so") next to the main library."""
    global BUILD, LIB
    if defines or out:
        tag = "_".join(d.replace("=", "") for d in defines) or "variant"
        BUILD, LIB = os.path.join(HERE, "_build_" + tag), os.path.join(HERE, out or f"libswe_{tag}.so")
    os.makedirs(BUILD, exist_ok=True)
    hdr = os.path.join(ROOT, "include", "swe.h")
    deps = [os.path.join(CSRC, d) for d in DEPS] + [hdr, __file__]
    objs = []
    for s in HOST_SRC:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        if force or _stale(obj, [src] + deps):
            cmd = ["g++", "-O2", "-fPIC", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-c", src, "-o", obj]
            subprocess.check_call(cmd)
        objs.append(obj)
    for s in CU_SRC:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        if force or _stale(obj, [src] + deps):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", *[f"-D{d}" for d in defines], "-I", _nccl_dirs()[0],
                   "-Xcompiler", "-fPIC,-ffp-contract=off",
                   "-Xptxas", "-v" if verbose else "-O3", "-c", src, "-o", obj]
            subprocess.check_call(cmd)
        objs.append(obj)
    if force or _stale(LIB, objs):
        inc, libdir = _nccl_dirs()
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-lcudart", "-L", libdir, "-l:libnccl.so.2",
               "-Xlinker", "-rpath=" + libdir]
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs))
