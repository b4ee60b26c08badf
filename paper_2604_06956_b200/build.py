"""Builds libnest.so (sm_100a) in-tree with nvcc.

One shared library from csrc/*.cu; links the NCCL and cuBLAS that the torch
wheel ships (the same libraries torch loads, so one NCCL / cuBLAS instance per
process).  Invoked by __graft_entry__.build() and by the tests on demand.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libnest.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _site_nvidia() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia wheel packages (nccl, cublas) not found")
    return list(spec.submodule_search_locations)[0]


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found")
    return p


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + \
        [os.path.join(ROOT, "include", "nest.h")]


STAMP = LIB + ".cmd"   # the nvcc command line libnest.so was built with


def _extra() -> list:
    # NEST_NVCC_EXTRA: extra -D flags for tuning builds (e.g. -DNEST_SEG_RANGE=128)
    return os.environ.get("NEST_NVCC_EXTRA", "").split()


def up_to_date() -> bool:
    """libnest.so is newer than every source AND was built with the default
    flags (a tuning build with NEST_NVCC_EXTRA writes a different stamp, so a
    later default build() replaces it instead of silently reusing it)."""
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return False
    if open(STAMP).read().strip() != " ".join(_extra()):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in sources() + headers() + [__file__])


def build(force: bool = False, verbose: bool = False, out: str = LIB) -> str:
    if not force and out == LIB and up_to_date():
        return LIB
    nv = _site_nvidia()
    nccl_inc, nccl_lib = os.path.join(nv, "nccl", "include"), os.path.join(nv, "nccl", "lib")
    cublas_inc, cublas_lib = os.path.join(nv, "cublas", "include"), os.path.join(nv, "cublas", "lib")
    tmp = out + ".tmp"
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "--extended-lambda",
           "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-shared",
           "-Xptxas", "-warn-spills",
           "-I", os.path.join(ROOT, "include"), "-I", nccl_inc, "-I", cublas_inc,
           *_extra(),
           *sources(),
           "-L", nccl_lib, "-L", cublas_lib, "-l:libnccl.so.2", "-l:libcublas.so.12", "-l:libcublasLt.so.12",
           "-Xlinker", f"-rpath={nccl_lib}:{cublas_lib}",
           "-o", tmp]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    r = subprocess.run(cmd, cwd=HERE, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr, file=sys.stderr)
    os.replace(tmp, out)
    if out == LIB:
        with open(STAMP, "w") as f:
            f.write(" ".join(_extra()))
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
