"""Shared test helpers (not a test module)."""
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def compile_c_example(out):
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if not gcc:
        pytest.skip("no gcc")
    lib = os.path.join(ROOT, "paper_2412_11614_b200")
    cmd = [gcc, "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "eta_c_abi.c"), "-L", lib, "-lisrs_egn", "-L",
           "/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath," + lib, "-lm", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


