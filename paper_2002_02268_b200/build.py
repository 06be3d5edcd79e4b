"""Build libelevate_b200.so in-tree with nvcc for sm_100a (no JIT cache).

`python -m paper_2002_02268_b200.build` or `__graft_entry__.build()`.
The .so is git-ignored but travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libelevate_b200.so")
SOURCES = ["elv_api.cu", "simt_gemm.cu", "tf32x3_gemm.cu", "stencil.cu", "host_pipeline.cu"]
HEADERS = ["elv_common.cuh", os.path.join("..", "..", "include", "elevate_b200.h")]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "-Xptxas", "-warn-spills",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = True, defines: tuple = (), out: str | None = None) -> str:
    """Compile SOURCES into `out` (default: the in-tree LIB).  `defines`
    (e.g. ("ELV_K7_PROF",)) produce instrumented tuning builds, which go to
    a separate path and are loaded with ELV_LIB=<path>."""
    target = out or LIB
    if not force and not defines and not _stale():
        return LIB
    objs = []
    build_dir = os.path.join(PKG, "_build" + ("_" + "_".join(defines).lower() if defines else ""))
    os.makedirs(build_dir, exist_ok=True)
    for s in SOURCES:
        obj = os.path.join(build_dir, s.replace(".cu", ".o"))
        cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(REPO, "include"), "-c",
               os.path.join(CSRC, s), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = target + ".tmp"
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs,
           "-o", tmp, "-ldl", "-lpthread"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print(LIB)
