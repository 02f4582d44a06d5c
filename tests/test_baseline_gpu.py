"""The BASELINE.json configs at FULL size on the B200, against the reference's
own outputs for the same runs (tests/golden/baseline_golden.json, produced by
tests/golden/make_baseline_golden.py from oracle/_ref = the reference headers):

  cfg1  256^2 x 1000 (the one-launch cluster path)
  cfg2  4096^2 x 100 000, slow-growth gene: ten checksums, one per 10 000
  cfg3  8192^2 image edge detection x 200 (through our PGM loader + typ=3 init)
  cfg4  the 4096-cell 128^2 x 5000 sweep: the labels CSV, byte for byte
  cfg5  32768^2 x 100 (periodic path and the fused peer-ring slab path)
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2102_10340_b200 as fhn

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD_PATH = os.path.join(HERE, "golden", "baseline_golden.json")


@pytest.fixture(scope="module")
def gold():
    if not os.path.exists(GOLD_PATH):
        pytest.skip("tests/golden/baseline_golden.json not generated")
    with open(GOLD_PATH) as f:
        return json.load(f)


def gene(g7):
    return fhn.Gene(dt=g7[0], a=g7[1], b=g7[2], eps=g7[3], c=g7[4], Du=g7[5], Dv=g7[6])


def digest(sim, rows, cols):
    return f"{int(sim.checksums()[0]):016x}"


def test_cfg1_256_x1000(gold):
    c = gold["cfg1"]
    with fhn.Simulator(256, 256, persistent=1) as sim:  # the cluster path, required
        sim.set_params(gene(c["gene7"]))
        sim.init(1, 42)
        assert int(sim.advance(c["iters"])[0]) == 0
        assert sim.launch_count() in (1, 4)  # one launch, or 3 rows-per-warp trials + the rest
        assert digest(sim, 256, 256) == c["checksum"]


def test_cfg2_4096_x100000(gold):
    c = gold["cfg2"]
    with fhn.Simulator(4096, 4096) as sim:
        sim.set_params(gene(c["gene7"]))
        sim.init(1, 42)
        for k, want in enumerate(c["checksums_every_10000"]):
            assert int(sim.advance(10000)[0]) == 0
            assert digest(sim, 4096, 4096) == want, f"after {(k + 1) * 10000} iterations"


def test_cfg3_8192_image_x200(gold, tmp_path):
    import importlib.util

    from paper_2102_10340_b200 import imageio

    spec = importlib.util.spec_from_file_location("make_baseline_golden",
                                                  os.path.join(HERE, "golden", "make_baseline_golden.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    cfg3_pixels = gen.cfg3_pixels

    c = gold["cfg3"]
    path = str(tmp_path / "cfg3.pgm")
    imageio.write_pgm(path, cfg3_pixels(c["rows"]))
    px = imageio.load_image_u8(path)
    with fhn.Simulator(c["rows"], c["cols"]) as sim:
        sim.set_params(gene(c["gene7"]))
        sim.init_image(px, c["ka"])
        assert c["init_checksum"] is None or digest(sim, c["rows"], c["cols"]) == c["init_checksum"]
        assert int(sim.advance(c["iters"])[0]) == c["bad_iter"]
        assert digest(sim, c["rows"], c["cols"]) == c["checksum"]


def test_cfg4_full_sweep_labels(gold):
    from paper_2102_10340_b200.engine import RunConfig
    from paper_2102_10340_b200.sweep import SweepSpec, sweep_grid

    c = gold["cfg4"]
    cfg = RunConfig()
    cfg.nn, cfg.nm = c["rows"], c["cols"]
    cfg.iter_max, cfg.nssp, cfg.seed = c["iter_max"], c["nssp"], c["seed"]
    spec = SweepSpec("du", list(np.linspace(0.02, 0.70, 64)), "dv", list(np.linspace(0.50, 1.20, 64)),
                     base_config=cfg)
    res = sweep_grid(spec)
    assert res.labels_csv.count("\n") == c["labels_csv_lines"]
    want_path = os.path.join(HERE, "golden", "cfg4_labels.csv")
    if os.path.exists(want_path):
        with open(want_path) as f:
            want = f.read()
        assert res.labels_csv == want
    assert hashlib.sha256(res.labels_csv.encode()).hexdigest() == c["labels_csv_sha256"]


def _cfg5_check(c, u, v):
    got = f"{fhn.checksum(fhn.GridState(c['rows'], c['cols'], u, v)):016x}"
    assert got == c["checksum"]


def test_cfg5_32768_x100_periodic(gold):
    c = gold["cfg5"]
    n = c["rows"]
    with fhn.Simulator(n, n) as sim:
        sim.set_params(gene(c["gene7"]))
        sim.init(2, 42)
        assert c["init_checksum"] is None or digest(sim, n, n) == c["init_checksum"]
        assert int(sim.advance(c["iters"])[0]) == c["bad_iter"]
        assert digest(sim, n, n) == c["checksum"]


def test_cfg5_32768_x100_slab_peer_ring(gold):
    """The same lattice through the multi-GPU code path (a world-1 fused peer
    ring: the torus row wrap through the neighbour-pointer jumps)."""
    from paper_2102_10340_b200.slab import SlabStepper

    c = gold["cfg5"]
    n = c["rows"]
    s = SlabStepper(n, n, rank=0, world=1, ghost=4, device=0)
    try:
        s.set_params(gene(c["gene7"]))
        s.init(2, 42)
        s.fill_ghosts()
        assert s.advance(c["iters"]) == c["bad_iter"]
        u, v = s.download()
    finally:
        s.close()
    _cfg5_check(c, u, v)


def test_cfg2_f64_4096_x1000(gold):
    """The reference's double instantiation on the cfg2 lattice (fp64 strict)."""
    if "cfg2_f64" not in gold:
        pytest.skip("fp64 entry not generated")
    c = gold["cfg2_f64"]
    with fhn.Simulator(c["rows"], c["cols"], precision="double") as sim:
        sim.set_params(gene(c["gene7"]))
        sim.init(1, 42)
        assert int(sim.advance(c["iters"])[0]) == c["bad_iter"]
        assert digest(sim, c["rows"], c["cols"]) == c["checksum"]
