"""The header-only C++ shim (include/sinkr/cuda/router.hpp) compiles against
the C-ABI (CPU) and runs a caller written against the reference API (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")


def _build(built_lib, out):
    libdir = os.path.dirname(built_lib)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           SRC, "-o", out, "-L", libdir, "-lsinkr_cuda", f"-Wl,-rpath,{libdir}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_shim_compiles(built_lib, tmp_path):
    _build(built_lib, str(tmp_path / "shim"))


@pytest.mark.gpu
def test_shim_runs(built_lib, tmp_path):
    exe = str(tmp_path / "shim")
    _build(built_lib, exe)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "shim OK" in res.stdout
