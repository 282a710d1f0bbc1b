"""The C ABI used from plain C++ (tests/cabi/example.cpp): compile with g++
against include/ and libgosma.so, then run on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_example(tmp_path, gosma):
    exe = tmp_path / "example"
    lib_dir = os.path.join(ROOT, "paper_1812_01232_b200")
    subprocess.check_call(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cabi", "example.cpp"), "-L", lib_dir,
                           "-lgosma", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)])
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr + out.stdout
    assert "cabi example ok" in out.stdout
