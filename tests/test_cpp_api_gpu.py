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


def _write_spec(path, d, keep_buffers=False):
    with open(path, "w") as f:
        f.write(f"x_param {d['x_param']}\ny_param {d['y_param']}\n")
        f.write("xs " + " ".join(repr(float(x)) for x in d["xs"]) + "\n")
        f.write("ys " + " ".join(repr(float(y)) for y in d["ys"]) + "\n")
        for k in ("nn", "nm", "iter_max", "nssp"):
            f.write(f"{k} {d[k]}\n")
        f.write(f"typ {d.get('typ', 1)}\nseed {d.get('seed', 42)}\n")
        f.write(f"per_cell_seed {int(d.get('per_cell_seed', False))}\nkeep_buffers {int(keep_buffers)}\n")


def _golden_sweeps():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)["sweeps"]


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(_golden_sweeps())))
def test_cpp_sweep_grid_equals_reference(i, tmp_path):
    """C++ sweep_grid<float> (sweep.hpp:249-326) on the batched device handle:
    the labels CSV equals the reference's own (tests/golden/golden.json), and
    with keep_buffers every cell's device statistics equal the host
    classify_outcome over its snapshot buffer."""
    case = _golden_sweeps()[i]
    spec = tmp_path / "spec.txt"
    _write_spec(spec, case["spec"], keep_buffers=True)
    r = subprocess.run([BIN, "--sweep", str(spec)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout == case["labels_csv"]
    assert " 0 mismatches" in r.stderr


@pytest.mark.gpu
def test_cpp_sweep_grid_cfg4_full_size(tmp_path):
    """BASELINE cfg4 through the C++ API: 64 x 64 (Du, Dv) cells of 128^2 x 5000,
    labels CSV byte-identical to the reference's (tests/golden/cfg4_labels.csv)."""
    import numpy as np
    spec = tmp_path / "cfg4.txt"
    _write_spec(spec, {"x_param": "du", "xs": list(np.linspace(0.02, 0.70, 64)), "y_param": "dv",
                       "ys": list(np.linspace(0.50, 1.20, 64)), "nn": 128, "nm": 128, "iter_max": 5000,
                       "nssp": 5, "seed": 42})
    r = subprocess.run([BIN, "--sweep", str(spec)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    with open(os.path.join(ROOT, "tests", "golden", "cfg4_labels.csv")) as f:
        assert r.stdout == f.read()
