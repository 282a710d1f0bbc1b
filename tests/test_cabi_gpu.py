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


GPU_BACKEND_TESTS = os.path.join(ROOT, "oracle", "_ref", "gpu_backend_tests")


@pytest.mark.skipif(not os.path.exists(GPU_BACKEND_TESTS),
                    reason="adapter not built (needs the reference headers: make -C oracle adapter)")
def test_reference_solver_cases_through_the_cpp_drop_in(gosma):
    """The compiled smalign::gpu adapter (adapter/smalign/gpu_backend.hpp)
    runs the reference's own solver test cases (test_solver.cpp:90-310) on the
    GPU: same inputs, same contract checks, FP64 reference bounds as the
    parity target of evaluate_branch_batch."""
    out = subprocess.run([GPU_BACKEND_TESTS], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
