"""Runs the reference's tests re-expressed against the C++ drop-in API
(tests/cpp/test_api.cpp over include/rdcnn/*.hpp -> librdcnn_cuda.so)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_api")


def test_cpp_api_builds():
    """CPU check: the drop-in headers compile and link against the C-ABI."""
    assert os.path.exists(BIN), "run __graft_entry__.build()"


@pytest.mark.gpu
def test_cpp_api_on_gpu():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
