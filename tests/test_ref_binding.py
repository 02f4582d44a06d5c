"""The reference-side FFI binding, compiled for real:
integration/reference_cuda_backend.patch adds a `cuda` BackendKind to the
reference's own headers (backend.hpp, kernels.hpp step() dispatch,
engine.hpp run/run_timed device-resident loops, a new cuda_backend.hpp over
include/rdcnn_cuda.h).  integration/Makefile applies it to a temporary copy
of /root/reference/proj/include and builds integration/ref_cuda_driver.cpp,
which runs the reference's acceptance criterion 1 (acceptance_main.cpp:76-100)
with cuda beside reference/blocked/parallel."""
import os
import shutil
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PATCH = os.path.join(ROOT, "integration", "reference_cuda_backend.patch")
BIN = os.path.join(ROOT, "integration", "_bin", "ref_cuda_driver")
REF_INCLUDE = "/root/reference/proj/include"


def test_patch_applies_to_a_copy_of_the_reference_headers():
    if not os.path.isdir(os.path.join(REF_INCLUDE, "rdcnn")):
        pytest.skip("reference tree absent (GPU box): the driver travels prebuilt")
    tmp = tempfile.mkdtemp()
    try:
        inc = os.path.join(tmp, "include")
        shutil.copytree(REF_INCLUDE, inc)
        r = subprocess.run(["patch", "-s", "-d", inc, "-p1", "-i", PATCH], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr
        backend = open(os.path.join(inc, "rdcnn", "backend.hpp")).read()
        kernels = open(os.path.join(inc, "rdcnn", "kernels.hpp")).read()
    finally:
        shutil.rmtree(tmp)
    # The reference keeps its CPU backends: the patch only adds a kind.
    assert "enum class BackendKind { Reference, Shift, Blocked, Parallel, Cuda };" in backend
    for name in ("reference", "shift", "blocked", "parallel", "cuda"):
        assert f'if (s == "{name}")' in backend
    for fn in ("kern::step_reference", "kern::step_blocked", "kern::step_parallel", "kern::step_shift",
               "cuda::step"):
        assert fn in kernels


def test_driver_built():
    assert os.path.exists(BIN), "run __graft_entry__.build()"


@pytest.mark.gpu
def test_reference_criterion1_with_cuda_beside_cpu_backends():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout
    lines = [l for l in r.stdout.splitlines() if l.startswith("criterion 1 ")]
    sums = {l.split()[2]: l.split()[3] for l in lines if "double" not in l}
    assert set(sums) == {"reference", "blocked", "parallel", "cuda"}
    assert set(sums.values()) == {"1026befcb693b1e5"}
