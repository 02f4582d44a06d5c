"""The C-ABI library (CPU-side checks: no kernel launches).

* librdcnn_cuda.so loads and exports every function include/rdcnn_cuda.h
  declares, and the ctypes binding covers exactly that set;
* host-side helpers (initial states, FNV digest, gene narrowing) equal the
  oracle bit for bit;
* argument validation mirrors the reference's error behaviour
  (backend.hpp:40-49, config.hpp:62-95, engine.hpp:57-61).
"""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2102_10340_b200 as fhn
from paper_2102_10340_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rdcnn_cuda.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(rdcnn_[a-z0-9_]+)\s*\(", text))


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def test_library_exports_every_declared_symbol():
    lib = fhn.load()
    names = declared_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert names == set(_lib.SIGNATURES), names ^ set(_lib.SIGNATURES)
    assert lib.rdcnn_abi_version() == 1


def test_library_is_sm100a_and_links_no_fallback():
    """The .so carries sm_100a SASS for the stencil kernels."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", fhn.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_host_init_equals_oracle(oracle):
    for typ, (r, c), seed in [(1, (11, 11), 77), (1, (64, 100), 42), (2, (3, 3), 1234), (2, (17, 23), 91),
                              (1, (256, 256), 42)]:
        ou, ov = oracle.init(typ, r, c, seed)
        s = fhn.init_center_square(r, c, seed) if typ == 1 else fhn.init_full_random(r, c, seed)
        assert np.array_equal(bits(s.u), bits(ou)) and np.array_equal(bits(s.v), bits(ov))
        assert fhn.checksum(s) == oracle.checksum(ou, ov)


def test_image_init_host(oracle):
    px = (np.arange(7 * 9, dtype=np.int64) * 37 % 256).astype(np.uint8).reshape(7, 9)
    for ka in (1.0, 0.3, 2.5):
        ou, ov = oracle.init_image(px, ka)
        s = fhn.init_from_image(px, fhn.Gene(ka=ka))
        assert np.array_equal(bits(s.u), bits(ou)) and np.array_equal(bits(s.v), bits(ov))


def test_params_narrowing(oracle):
    g = fhn.Gene(a=-0.05, b=1.3, eps=-0.1, c=1.0, Du=0.06, Dv=1.0, dt=0.1)
    p = fhn.params_from_gene(g)
    want = oracle.params(g.to_vector())
    got = np.array([p.dt, p.a, p.b, p.eps, p.c, p.du, p.dv], np.float32)
    assert np.array_equal(bits(got), bits(want))


def test_checksum_known_answer():
    s = fhn.init_center_square(256, 256, 42)
    assert fhn.checksum_hex(fhn.checksum(s)) == f"{fhn.checksum(s):016x}"
    assert fhn.checksum(s) != fhn.checksum(fhn.init_center_square(256, 256, 43))


def test_invalid_arguments_fail_loudly():
    lib = fhn.load()
    h = ctypes.c_void_p()
    assert lib.rdcnn_sim_create(2, 5, 1, 0, 0, ctypes.byref(h)) == 1
    assert "3x3" in _lib.last_error()
    assert lib.rdcnn_sim_create(8, 8, 0, 0, 0, ctypes.byref(h)) == 1
    assert lib.rdcnn_sim_create(8, 8, 1, 0, 7, ctypes.byref(h)) == 1
    assert lib.rdcnn_slab_create(8, 8, 3, 0, 0, ctypes.byref(h)) == 1
    assert lib.rdcnn_slab_create(4, 8, 4, 0, 0, ctypes.byref(h)) == 1
    assert lib.rdcnn_sim_advance(None, 1, None) == 1
    assert lib.rdcnn_init_center_square_host(10, 40, 1, None, None) == 1


def test_backend_selection_mirrors_reference():
    assert fhn.make_backend("cuda").kind == "cuda"
    for name in ("reference", "parallel", "blocked", "shift"):
        with pytest.raises(ValueError, match="CPU backend"):
            fhn.make_backend(name)
    with pytest.raises(ValueError, match="unknown backend"):
        fhn.make_backend("gpu")
    with pytest.raises(ValueError):
        fhn.make_backend("cuda", tile_rows=0)
    with pytest.raises(ValueError):
        fhn.make_backend("cuda", threads=-1)


def test_validate_config_reports_every_issue():
    g = fhn.Gene(dt=-1.0)
    kinds = [i.split(":")[0] for i in fhn.validate_config(fhn.RunConfig(nn=2, nm=2, iter_max=10, nssp=3), g)]
    assert kinds == ["InvalidSize", "InvalidSize", "InvalidSchedule", "NonFiniteGene"]
    kinds = [i.split(":")[0] for i in fhn.validate_config(fhn.RunConfig(init_mode=3, nssp=0), fhn.Gene())]
    assert kinds == ["InvalidSchedule", "MissingImage"]
    assert fhn.validate_config(fhn.RunConfig(), fhn.Gene()) == []


def test_run_rejects_bad_schedule_and_shape_before_touching_the_device():
    with pytest.raises(fhn.ScheduleError):
        fhn.run(fhn.RunConfig(nn=16, nm=16, iter_max=100, nssp=3), fhn.Gene(), fhn.init_center_square(16, 16, 1))
    with pytest.raises(ValueError):
        fhn.run(fhn.RunConfig(nn=16, nm=16, iter_max=10, nssp=1), fhn.Gene(), fhn.init_center_square(32, 32, 1))


def test_no_gpu_means_loud_failure():
    """Without a usable device the product raises; it never falls back."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.RdcnnError) as e:
        fhn.Simulator(16, 16)
    assert e.value.code == 3


def test_batch_gene_narrowing_equals_c_abi():
    """Simulator.set_params narrows batches of genes with numpy (one pass);
    it must equal the C-ABI's per-gene make_params<float> narrowing
    (rdcnn_params_from_gene, model.hpp:24-32) bit for bit."""
    import numpy as np

    import paper_2102_10340_b200 as fhn
    from paper_2102_10340_b200.engine import ParamsF32, params_from_gene

    rng = np.random.default_rng(7)
    genes = [fhn.Gene(a=float(rng.normal()), b=float(rng.normal()), eps=float(rng.normal() * 0.1),
                      c=float(rng.normal()), Du=float(abs(rng.normal())), Dv=float(abs(rng.normal())),
                      dt=float(abs(rng.normal()) * 0.1)) for _ in range(500)]
    genes += [fhn.Gene(Du=x) for x in np.linspace(0.02, 0.70, 64)]
    from paper_2102_10340_b200.engine import ParamsF64, gene_batch

    fields = [f for f, _ in ParamsF32._fields_]
    ref = np.array([[getattr(params_from_gene(g), f) for f in fields] for g in genes], np.float32)
    assert fields == ["dt", "a", "b", "eps", "c", "du", "dv"]
    # The helper Simulator.set_params passes to rdcnn_sim_set_params: a ctypes
    # ParamsF32 array over the numpy buffer, read back struct by struct.
    batch = gene_batch(genes)
    assert len(batch) == len(genes) and isinstance(batch[0], ParamsF32)
    got = np.array([[getattr(batch[k], f) for f in fields] for k in range(len(genes))], np.float32)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
    b64 = gene_batch(genes, "double")
    assert isinstance(b64[0], ParamsF64)
    got64 = np.array([[getattr(b64[k], f) for f in fields] for k in range(len(genes))])
    assert np.array_equal(got64, np.array([g.to_vector() for g in genes]))


# The C++ drop-in headers mirror the reference's: each one compiles on its
# own (its include graph is complete), as a reference translation unit that
# includes only, say, rdcnn/kernels.hpp expects.
HEADERS = ["gene", "grid", "rng", "model", "backend", "config", "init", "kernels", "engine", "bench", "sweep",
           "cuda_api"]


@pytest.mark.parametrize("name", HEADERS)
def test_cpp_header_compiles_standalone(tmp_path, name):
    import shutil
    import subprocess
    cxx = shutil.which("g++")
    if cxx is None:
        pytest.skip("no g++")
    src = tmp_path / f"t_{name}.cpp"
    src.write_text(f'#include "rdcnn/{name}.hpp"\nint main() {{ return 0; }}\n')
    r = subprocess.run([cxx, "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
