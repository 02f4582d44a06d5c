"""fp64 path (§8f3): the reference templates instantiate double throughout
(grid.hpp:13-28, model.hpp:24-32 make_params<double>); the device kernel
must reproduce them bit for bit in strict mode."""
import ctypes
import json
import os

import numpy as np
import pytest

import paper_2102_10340_b200 as fhn

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def gene_from7(g7):
    return fhn.Gene(dt=g7[0], a=g7[1], b=g7[2], eps=g7[3], c=g7[4], Du=g7[5], Dv=g7[6])


@pytest.fixture(scope="module")
def cases_f64():
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)["cases_f64"]


def test_div3_f64_on_device():
    lib = fhn.load()
    n, first = ctypes.c_uint64(), ctypes.c_uint64()
    assert lib.rdcnn_selftest_div3_f64(0, 1 << 30, ctypes.byref(n), ctypes.byref(first)) == 0
    assert n.value == 0, hex(first.value)


@pytest.mark.parametrize("levels", (1, 2, 4))
def test_golden_f64(cases_f64, levels):
    for c in cases_f64:
        r, k = c["rows"], c["cols"]
        with fhn.Simulator(r, k, levels=levels, precision="double") as sim:
            sim.set_params(gene_from7(c["gene7"]))
            sim.init(c["typ"], c["seed"])
            u0, v0 = sim.download()
            assert f"{fhn.checksum(fhn.GridState(r, k, u0, v0)):016x}" == c["init_checksum"], c["name"]
            bad = sim.advance(c["iters"])
            assert int(bad[0]) == c["bad_iter"], (c["name"], levels)
            if c["bad_iter"] == 0:
                u, v = sim.download()
                assert f"{fhn.checksum(fhn.GridState(r, k, u, v)):016x}" == c["checksum"], (c["name"], levels)


@pytest.mark.parametrize("rows,cols", [(3, 3), (5, 7), (17, 23), (64, 64), (33, 130), (40, 126), (96, 512)])
def test_random_shapes_f64(oracle, rows, cols):
    u0, v0 = oracle.init_f64(2, rows, cols, 77 + rows + cols)
    ou, ov, bad = oracle.run_f64(rows, cols, u0, v0, 19)
    assert bad == 0
    for levels in (1, 2, 4):
        with fhn.Simulator(rows, cols, levels=levels, precision="double") as sim:
            sim.upload(u0, v0)
            assert int(sim.advance(19)[0]) == 0
            u, v = sim.download()
        assert np.array_equal(bits(u), bits(ou)) and np.array_equal(bits(v), bits(ov)), (rows, cols, levels)


def test_f64_batch_and_api(oracle):
    genes = [fhn.Gene(Du=0.3, Dv=1.0), fhn.Gene(dt=100.0), fhn.Gene(a=-0.05)]
    u0, v0 = oracle.init_f64(1, 24, 40, 42)
    with fhn.Simulator(24, 40, batch=3, levels=4, precision="double") as sim:
        sim.set_params(genes)
        sim.init(1, 42)
        bad = sim.advance(37)
        u, v = sim.download()
    for k, g in enumerate(genes):
        ou, ov, obad = oracle.run_f64(24, 40, u0, v0, 37, g.to_vector())
        assert int(bad[k]) == obad
        fin = np.isfinite(ou) & np.isfinite(ov)
        assert np.array_equal(bits(u.reshape(3, -1)[k])[fin], bits(ou)[fin])
    # reference-shaped API in double
    st = fhn.init_center_square(64, 64, 42, precision="double")
    out = fhn.run(fhn.RunConfig(nn=64, nm=64, iter_max=200, nssp=5, precision="double"), fhn.Gene(), st)
    ou, ov, _ = oracle.run_f64(64, 64, st.u, st.v, 200)
    assert np.array_equal(bits(out.final_state.u), bits(ou))
