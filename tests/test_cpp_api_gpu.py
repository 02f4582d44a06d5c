"""Runs the reference's tests re-expressed against the C++ drop-in API
(tests/cpp/test_api.cpp over include/rdcnn/*.hpp -> librdcnn_cuda.so)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_api")
SEAM = os.path.join(ROOT, "tests", "cpp", "test_model_seam")


def test_cpp_api_builds():
    """CPU check: the drop-in headers compile and link against the C-ABI."""
    assert os.path.exists(BIN), "run __graft_entry__.build()"


@pytest.mark.gpu
def test_cpp_api_on_gpu():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_model_seam_builds():
    """CPU check: a CellModel translation unit compiles with nvcc against the headers."""
    assert os.path.exists(SEAM), "run __graft_entry__.build()"


@pytest.mark.gpu
def test_model_seam_on_gpu():
    """The CellModel seam (model.hpp:13-21) on the device: the reference's
    pure-diffusion mass test, exact order vs a host loop, a user-written FHN
    model == the built-in kernels, non-finite detection."""
    r = subprocess.run([SEAM], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_cpp_bench_emitters_host():
    """CPU: bench.hpp's emit_csv / emit_table / emit_json formats on the drop-in
    API (test_bench.cpp cases), no device work."""
    r = subprocess.run([BIN, "--host-only"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout
