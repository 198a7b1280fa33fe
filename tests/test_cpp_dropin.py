"""Builds tests/cpp/dropin_test.cpp against the C++ drop-in header and runs it on the GPU.

The C++ test restates the reference's own transform/params test cases
(proj/tests/transform_test.cpp, params_test.cpp) through nttk_gpu/nttk.hpp, i.e. through
the C ABI of libnttk_gpu.so, exactly as a C++ user of the reference would call it."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2402_00675_b200")


def build(out):
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", f"-I{PKG}/include",
           os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp"), f"-L{PKG}", "-lnttk_gpu",
           f"-Wl,-rpath,{PKG}", "-o", out]
    subprocess.run(cmd, check=True)


def test_dropin_header_compiles(tmp_path):
    """CPU: the drop-in header + C ABI link cleanly (no GPU needed to build)."""
    build(str(tmp_path / "dropin_test"))


@pytest.mark.gpu
def test_dropin_reference_cases_on_gpu(tmp_path):
    exe = str(tmp_path / "dropin_test")
    build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
