"""Pins the CPU oracle (oracle/fhn_oracle.c) before anything is checked
against it: the reference's known answers, the reference's own code
(oracle/_ref) on the golden fixtures, and the model KATs of
test_model.cpp / test_kernels.cpp.  CPU only."""
import ctypes
import os

import numpy as np
import pytest

from oracle.oracle import DEFAULT_GENE7, REF_SO

HAVE_REF = os.path.exists(REF_SO)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


# --- known answers recorded by the reference (proj/test_output.txt) -----------

def test_kat_criterion1_checksum(oracle):
    """256^2 typ=1 seed 42, 1000 iterations: 1026befcb693b1e5 (test_output.txt:8)."""
    u, v = oracle.init(1, 256, 256, 42)
    u, v, bad = oracle.run(256, 256, u, v, 1000)
    assert bad == 0
    assert oracle.checksum(u, v) == 0x1026BEFCB693B1E5


def test_kat_criterion10_checksum(oracle):
    """64^2 typ=1 seed 42, 200 iterations: ced829150965fba9 (test_output.txt:23)."""
    u, v = oracle.init(1, 64, 64, 42)
    u, v, bad = oracle.run(64, 64, u, v, 200)
    assert bad == 0 and oracle.checksum(u, v) == 0xCED829150965FBA9


def test_kat_blowup_iteration(oracle):
    """dt=100 on 16^2 typ=1 seed 42 blows up at iteration 4 (test_engine.cpp:95)."""
    g = list(DEFAULT_GENE7)
    g[0] = 100.0
    u, v = oracle.init(1, 16, 16, 42)
    _, _, bad = oracle.run(16, 16, u, v, 1000, g)
    assert bad == 4


# --- golden fixtures produced by the reference itself ---------------------------

def test_golden_cases(oracle, golden):
    for c in golden:
        u, v = oracle.init(c["typ"], c["rows"], c["cols"], c["seed"])
        assert f"{oracle.checksum(u, v):016x}" == c["init_checksum"], c["name"]
        u, v, bad = oracle.run(c["rows"], c["cols"], u, v, c["iters"], c["gene7"])
        assert bad == c["bad_iter"], c["name"]
        if bad == 0:
            assert f"{oracle.checksum(u, v):016x}" == c["checksum"], c["name"]


def test_golden_cases_f64(oracle):
    """fp64 digests from the reference (make_params<double>, no narrowing)."""
    import json
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(os.path.join(root, "tests", "golden", "golden.json")) as f:
        cases = json.load(f)["cases_f64"]
    for c in cases:
        u, v = oracle.init_f64(c["typ"], c["rows"], c["cols"], c["seed"])
        assert f"{oracle.checksum(u, v):016x}" == c["init_checksum"], c["name"]
        u, v, bad = oracle.run_f64(c["rows"], c["cols"], u, v, c["iters"], c["gene7"])
        assert bad == c["bad_iter"], c["name"]
        if bad == 0:
            assert f"{oracle.checksum(u, v):016x}" == c["checksum"], c["name"]


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (reference tree absent)")
def test_oracle_equals_reference_code():
    """The C restatement and the reference headers agree bit for bit, including
    the post-blow-up finite cells and on every exact-order backend."""
    from oracle.oracle import Oracle, Reference
    o, r = Oracle(), Reference()
    for rows, cols, typ, seed, iters in [(17, 23, 2, 91, 20), (32, 48, 2, 1001, 25), (40, 13, 2, 3, 9),
                                         (64, 64, 1, 42, 200)]:
        u0, v0 = o.init(typ, rows, cols, seed)
        ru, rv = r.init(typ, rows, cols, seed)
        assert np.array_equal(bits(u0), bits(ru)) and np.array_equal(bits(v0), bits(rv))
        ou, ov, _ = o.run(rows, cols, u0, v0, iters)
        for be in ("reference", "blocked", "parallel"):
            fu, fv, bad, _ = r.run_timed(rows, cols, u0, v0, iters, backend=be)
            assert bad == 0
            assert np.array_equal(bits(fu), bits(ou)) and np.array_equal(bits(fv), bits(ov)), be


# --- model and stencil known answers (test_model.cpp, test_kernels.cpp) --------

def test_reaction_kats(oracle):
    L = oracle.L
    p32 = oracle.params()
    p64 = np.asarray(DEFAULT_GENE7, np.float64)
    ptr32 = p32.ctypes.data_as(ctypes.c_void_p)
    ptr64 = p64.ctypes.data_as(ctypes.c_void_p)
    assert abs(L.orc_reaction_u_f32(1.0, 0.0, ptr32) - 0.6666667) <= 1e-6 * 0.6666667
    assert abs(L.orc_reaction_u_f64(1.0, 0.0, ptr64) - 2.0 / 3.0) <= 1e-15
    assert abs(L.orc_reaction_v_f64(0.0, 0.0, ptr64) - (-0.03)) <= 1e-12 * 0.03
    assert abs(L.orc_reaction_v_f64(1.0, 0.0, ptr64) - 0.07) <= 1e-12 * 0.07
    un, vn = ctypes.c_double(), ctypes.c_double()
    L.orc_cell_update_f64(1.0, 0.0, 0.0, 0.0, ptr64, ctypes.byref(un), ctypes.byref(vn))
    assert abs(un.value - 1.0666667) <= 1e-7 * 1.0666667 and abs(vn.value - 0.007) <= 1e-12
    L.orc_cell_update_f64(0.0, 0.0, 0.0, 0.0, ptr64, ctypes.byref(un), ctypes.byref(vn))
    assert un.value == 0.0 and abs(vn.value - (-0.003)) <= 1e-12 * 0.003


def test_reaction_u_odd(oracle):
    rng = np.random.default_rng(11)
    p = oracle.params()
    ptr = p.ctypes.data_as(ctypes.c_void_p)
    for u, v in rng.uniform(-2, 2, (200, 2)).astype(np.float32):
        a = oracle.L.orc_reaction_u_f32(float(-u), float(-v), ptr)
        b = oracle.L.orc_reaction_u_f32(float(u), float(v), ptr)
        assert np.float32(a) == -np.float32(b)


def test_laplacian_delta_3x3(oracle):
    layer = np.zeros(9, np.float64)
    layer[4] = 1.0
    f = oracle.L.orc_laplacian5_f64
    ptr = layer.ctypes.data_as(ctypes.c_void_p)
    assert f(ptr, 3, 3, 1, 1) == -4.0
    for i, j in [(0, 1), (1, 0), (1, 2), (2, 1)]:
        assert f(ptr, 3, 3, i, j) == 1.0
    for i, j in [(0, 0), (0, 2), (2, 0), (2, 2)]:
        assert f(ptr, 3, 3, i, j) == 0.0


def test_stencil_support_after_one_step(oracle):
    """test_kernels.cpp:98-118: u differs on 5 cells, v on 1."""
    z = np.zeros(256, np.float32)
    pu = z.copy()
    pu[8 * 16 + 8] = 1.0
    bu, bv, _ = oracle.run(16, 16, z, z, 1)
    hu, hv, _ = oracle.run(16, 16, pu, z, 1)
    assert int((bits(bu) != bits(hu)).sum()) == 5
    assert int((bits(bv) != bits(hv)).sum()) == 1


def test_rng_stream_order(oracle):
    """test_rng_init.cpp:53-58: u layer first, then v, row-major; 11x11 typ=1 == typ=2."""
    u1, v1 = oracle.init(1, 11, 11, 77)
    u2, v2 = oracle.init(2, 11, 11, 77)
    assert np.array_equal(bits(u1), bits(u2)) and np.array_equal(bits(v1), bits(v2))
    u, v = oracle.init(2, 3, 3, 1234)
    f = oracle.L.orc_rng_u64
    f.restype = ctypes.c_uint64
    f.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
    draws = [np.float32(np.float32(f(1234, k) >> 40) * np.float32(2.0 ** -24)) for k in range(18)]
    assert np.array_equal(bits(np.concatenate([u, v])), bits(np.array(draws, np.float32)))


def test_center_square_geometry(oracle):
    u, v = oracle.init(1, 512, 512, 42)
    U = u.reshape(512, 512)
    mask = np.zeros((512, 512), bool)
    mask[250:261, 250:261] = True
    assert (U[~mask] == 0).all() and (v.reshape(512, 512)[~mask] == 0).all()
    assert 100 < int((U[mask] != 0).sum()) <= 121


# --- the divide-by-3 proof the product kernel relies on -----------------------

def test_div3_exhaustive_cpu(oracle):
    """All 2^32 fp32 inputs: the corrected-reciprocal quotient equals IEEE x/3
    except at x = -0.0 (sign of zero), which u*u never produces."""
    n, first = oracle.div3_sweep()
    assert (n, first) == (1, 0x80000000)


def test_div3_two_op_gate_cpu(oracle):
    """The gated 2-op x/3 of the strict fp32 kernel (fhn_stencil.cuh div3_rn2),
    over every x >= +0: the raw quotient differs from IEEE x/3 only on
    [2^-125, 2^-123]; the composite RN(c - x/3) of model.hpp:39 is identical
    for c = +-2^-90 (the gate) and c = 1 on every input."""
    n, lo, hi = oracle.div3_two_op_sweep(0)
    assert n == 5592406
    assert lo == 0x01000000 and hi == 0x02000000  # 2^-125 .. 2^-123
    n, lo, hi = oracle.div3_two_op_sweep(1)
    assert n == 0, (n, hex(lo), hex(hi))


def test_baseline_golden_fixture_consistent(oracle):
    """tests/golden/baseline_golden.json (the reference's own full-size runs
    of the BASELINE configs, replayed on the B200 by test_baseline_gpu.py):
    cfg1 is the recorded criterion-1 KAT; the cfg4 CSV matches its digest;
    the C oracle reproduces the first cfg2 checkpoint's prefix cheaply
    (1000 iterations of 512^2 of the same gene is covered by golden.json)."""
    import hashlib
    import json

    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    path = os.path.join(here, "baseline_golden.json")
    if not os.path.exists(path):
        pytest.skip("baseline golden not generated")
    with open(path) as f:
        g = json.load(f)
    assert g["cfg1"]["checksum"] == "1026befcb693b1e5"  # test_output.txt:8
    if "cfg2" in g:
        assert len(g["cfg2"]["checksums_every_10000"]) == 10
    if "cfg4" in g:
        with open(os.path.join(here, "cfg4_labels.csv")) as f:
            csv = f.read()
        assert hashlib.sha256(csv.encode()).hexdigest() == g["cfg4"]["labels_csv_sha256"]
        assert csv.startswith("x_value,y_value,label,")
        assert csv.count("\n") == g["cfg4"]["labels_csv_lines"] == 4097
