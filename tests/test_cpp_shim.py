"""The C++ drop-in (include/comerge/cuda.hpp): built in-tree by `make`,
compiled check on CPU, the reference's unit-test cases replayed on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "shim_test")


def test_shim_test_binary_is_built():
    assert os.path.exists(BIN), "run `make` (builds tests/cpp/shim_test)"
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libcomerge_cuda.so" in out


@pytest.mark.gpu
def test_cpp_shim_on_gpu():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout
