"""Build recipe for the in-tree CUDA library (sm_100a only).

``python -m paper_2604_16883_b200.build`` or ``__graft_entry__.build()``
compiles ``csrc/*.cu`` with nvcc into ``_lib/libsinkr_cuda.so``.  The library
travels with the repo snapshot to the GPU box; nothing is JIT-compiled there.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIB_DIR, "libsinkr_cuda.so")
# bench support (tools/e2e_timer.cpp): a C++ caller's timed decode loop
BENCH_LIB = os.path.join(LIB_DIR, "libsinkr_bench.so")
TOOLS = os.path.join(HERE, "tools")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a library")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cuh", ".h", ".hpp", ".cpp")))


def translation_units():
    """engine.cu (device kernels + the engine) and the host-only C++ units
    (calibration, snapshots, analysis) — all linked into one library."""
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    deps = sources() + [os.path.join(ROOT, "include", "sinkr_cuda.h")]
    return all(os.path.getmtime(p) <= t for p in deps)


def build_bench_lib(force: bool = False) -> str:
    src = os.path.join(TOOLS, "e2e_timer.cpp")
    if (not force and os.path.exists(BENCH_LIB) and os.path.exists(LIB)
            and os.path.getmtime(BENCH_LIB) >= max(os.path.getmtime(src), os.path.getmtime(LIB))):
        return BENCH_LIB
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I", os.path.join(ROOT, "include"), src,
           "-L", LIB_DIR, "-lsinkr_cuda", "-Wl,-rpath,$ORIGIN", "-o", BENCH_LIB + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("g++ failed:\n" + res.stdout + res.stderr)
    os.replace(BENCH_LIB + ".tmp", BENCH_LIB)
    return BENCH_LIB


def build_library(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        build_bench_lib()
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    cmd = [nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo",
           # host side: no FMA contraction, so tau(L) matches the reference
           "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
           "-Xptxas", "-v" if verbose else "-O3",
           "-shared", "-I", os.path.join(ROOT, "include"),
           *translation_units(), "-o", LIB + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(LIB + ".tmp", LIB)
    build_bench_lib(force=True)
    return LIB


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose="-v" in sys.argv))
