"""The C++ host layer (include/stk_gpu.hpp) compiles against the C ABI library and, on a
GPU, passes its reference-named tests (tests/cpp/test_stk_gpu.cpp)."""
import subprocess

import pytest

from conftest import ROOT

BIN = ROOT / "tests" / "cpp" / "test_stk_gpu"


def build_cpp_test():
    import paper_1912_10082_b200._lib  # noqa: F401  (ensures the .so is built)
    pkg = ROOT / "paper_1912_10082_b200"
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", f"-I{ROOT / 'include'}",
           str(ROOT / "tests" / "cpp" / "test_stk_gpu.cpp"), "-o", str(BIN), f"-L{pkg}",
           "-l:_stk_gpu.so", f"-Wl,-rpath,{pkg}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return BIN


def test_cpp_host_layer_compiles():
    build_cpp_test()


@pytest.mark.gpu
def test_cpp_host_layer_runs_on_gpu():
    b = build_cpp_test()
    r = subprocess.run([str(b)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL OK" in r.stdout
