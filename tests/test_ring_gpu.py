"""The in-process multi-device ring (rdcnn_ring_*, slab.Ring) on the B200.

The pool gives one GPU, so every ring here puts all its slabs on device 0:
the slabs' blocks run interleaved on one stream and their edge warps read
each other's rows through the same peer-pointer code path that crosses
NVLink on a multi-GPU box.  Checked bit for bit against:

* the C oracle (periodic torus, the reference algorithm) on small lattices,
  including uneven slabs, every fusion depth and blow-ups placed on slab
  edges (the reference's exact iteration, engine.hpp:79);
* the reference's own digest of BASELINE configs[4] (32768^2 x 100,
  tests/golden/baseline_golden.json) at N = 2, 4 and 8 slabs -- the
  decomposition the 8-GPU scaling run uses.
"""
import json
import os

import numpy as np
import pytest

import paper_2102_10340_b200 as fhn
from paper_2102_10340_b200.slab import Ring

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
DEFAULT_G7 = [0.1, -0.3, 1.3, -0.1, 1.0, 0.06, 1.0]


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def gene7(g7):
    return fhn.Gene(dt=g7[0], a=g7[1], b=g7[2], eps=g7[3], c=g7[4], Du=g7[5], Dv=g7[6])


@pytest.fixture(scope="module")
def orc():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.mark.parametrize("n,rows,cols,ghost,levels,iters", [
    (2, 64, 96, 4, 4, 53),
    (3, 99, 128, 4, 4, 61),      # uneven slabs (33 rows each)
    (4, 102, 64, 4, 2, 40),      # uneven: 26, 26, 25, 25
    (4, 96, 257, 4, 4, 37),      # odd column count (W=1 lanes)
    (5, 160, 128, 8, 8, 70),     # full-width bands (kWrap), ghost 8
    (8, 128, 96, 4, 1, 19),
    (1, 48, 64, 4, 4, 33),       # world 1: the ring closes on itself
])
def test_ring_equals_oracle(orc, n, rows, cols, ghost, levels, iters):
    u0, v0 = orc.init(2, rows, cols, 7)
    ou, ov, obad = orc.run(rows, cols, u0, v0, iters, DEFAULT_G7)
    assert obad == 0
    with Ring(rows, cols, [0] * n, ghost=ghost, levels=levels) as ring:
        ring.upload(u0, v0)
        assert int(ring.advance(iters)[0]) == 0
        u, v = ring.download()
        # A second call continues from the device state.
        assert int(ring.advance(5)[0]) == 0
        u2, v2 = ring.download()
    assert np.array_equal(bits(u), bits(ou)) and np.array_equal(bits(v), bits(ov))
    pu, pv, _ = orc.run(rows, cols, ou, ov, 5, DEFAULT_G7)
    assert np.array_equal(bits(u2), bits(pu)) and np.array_equal(bits(v2), bits(pv))


def test_ring_init_matches_global_init(orc):
    """rdcnn_ring_init builds each slab as rows of the global lattice."""
    for typ in (1, 2):
        with Ring(90, 64, [0, 0, 0], ghost=4) as ring:
            ring.init(typ, 42)
            u, v = ring.download()
        ou, ov = orc.init(typ, 90, 64, 42)
        assert np.array_equal(bits(u), bits(ou)) and np.array_equal(bits(v), bits(ov))


def _blowup_state(orc, rows, cols, r, c, amp):
    u0, v0 = orc.init(2, rows, cols, 3)
    u0 = u0.copy()
    u0[r * cols + c] = np.float32(amp)
    return u0, v0


@pytest.mark.parametrize("n,row", [(4, 23), (4, 24), (4, 0), (3, 47), (2, 31)])
# Seed amplitudes whose blow-up lands at iterations 4, 5, 7-8 and 9-10 (or
# never, for some placements): first levels of blocks and mid-block levels.
@pytest.mark.parametrize("amp", [40.0, 9.28730297088623, 7.935965061187744, 7.889298439025879])
def test_ring_blowup_exact_iteration_on_slab_edges(orc, n, row, amp):
    """A blow-up seeded on (or next to) a slab edge: the ring reports the
    oracle's iteration and leaves the post-blow-up state, every finite cell
    bit-identical and the same cells non-finite."""
    rows, cols = 96 if n != 3 else 99, 64
    u0, v0 = _blowup_state(orc, rows, cols, row, 17, amp)
    ou, ov, obad = orc.run(rows, cols, u0, v0, 60, DEFAULT_G7)
    with Ring(rows, cols, [0] * n, ghost=4) as ring:
        ring.upload(u0, v0)
        bad = int(ring.advance(60)[0])
        u, v = ring.download()
    assert bad == obad
    # The oracle stops at its first bad iteration too (run_timed semantics).
    assert np.array_equal(np.isfinite(u), np.isfinite(ou)) and np.array_equal(np.isfinite(v), np.isfinite(ov))
    fu, fv = np.isfinite(ou), np.isfinite(ov)
    assert np.array_equal(bits(u)[fu], bits(ou)[fu]) and np.array_equal(bits(v)[fv], bits(ov)[fv])


def test_ring_blowup_split_calls_and_block_granularity(orc):
    rows, cols = 96, 64
    u0, v0 = _blowup_state(orc, rows, cols, 24, 17, 7.889298439025879)
    _, _, obad = orc.run(rows, cols, u0, v0, 60, DEFAULT_G7)
    assert obad == 9
    # Split: the first call stays finite, the second reports its own offset.
    with Ring(rows, cols, [0] * 4, ghost=4) as ring:
        ring.upload(u0, v0)
        assert int(ring.advance(obad - 2)[0]) == 0
        assert int(ring.advance(10)[0]) == 2
    # exact=False: the first iteration of the first bad block (block of 4).
    with Ring(rows, cols, [0] * 4, ghost=4, exact=False) as ring:
        ring.upload(u0, v0)
        got = int(ring.advance(60)[0])
    assert got == ((obad - 1) // 4) * 4 + 1


def test_ring_trace_block_reports_edge_waits_and_peer_bytes():
    rows, cols, n, k = 512, 1024, 4, 4
    with Ring(rows, cols, [0] * n, ghost=4) as ring:
        ring.init(2, 1)
        ring.advance(8)
        tr = ring.trace_block(k)
    assert tr.shape[1] == 6 and len(tr) > 0
    slab, t0, t1, smid, wait, peer = (tr[:, i] for i in range(6))
    assert set(slab.tolist()) == set(range(n))
    assert (t1 >= t0).all() and (smid < 148).all()
    edge = peer > 0
    # Every slab reads k rows above and k rows below from its neighbours,
    # for every column band: 2*k rows x cols x 2 planes x 4 bytes in total
    # (halo lanes included: bands overlap by their halo).
    for r in range(n):
        per = peer[slab == r]
        assert per.sum() >= 2 * k * cols * 2 * 4
        assert (per > 0).sum() >= 2
    assert (wait[~edge] == 0).all()


def test_ring_matches_periodic_on_4096(orc):
    """cfg2 lattice: 4 slabs on one device == the periodic single-handle run."""
    g7 = [0.1, -0.05, 1.3, -0.1, 1.0, 0.06, 1.0]
    with fhn.Simulator(4096, 4096) as sim:
        sim.set_params(gene7(g7))
        sim.init(1, 42)
        sim.advance(400)
        want = sim.checksums()[0]
    with Ring(4096, 4096, [0] * 4, ghost=4) as ring:
        ring.set_params(gene7(g7))
        ring.init(1, 42)
        assert int(ring.advance(400)[0]) == 0
        u, v = ring.download()
    assert fhn.checksum(fhn.GridState(4096, 4096, u, v)) == int(want)


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(HERE, "golden", "baseline_golden.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_cfg5_32768_x100_ring_n_slabs(gold, n):
    """BASELINE configs[4] decomposed exactly as the N-GPU run decomposes it
    (N row slabs, fused peer exchange), all on device 0: the reference's own
    digest of the 32768^2 x 100 run."""
    c = gold["cfg5"]
    size = c["rows"]
    with Ring(size, size, [0] * n, ghost=4) as ring:
        ring.set_params(gene7(c["gene7"]))
        ring.init(2, 42)
        assert int(ring.advance(c["iters"])[0]) == c["bad_iter"]
        assert ring.launch_count() == n * (c["iters"] // 4)
        u, v = ring.download()
    got = f"{fhn.checksum(fhn.GridState(size, size, u, v)):016x}"
    assert got == c["checksum"]


def test_cfg5_sized_ring_blowup_crossing_slabs():
    """A blow-up seeded on the slab edge of an 8-slab 32768^2 ring: the ring
    reports the same iteration as the periodic single-handle run of the same
    state, and the post-blow-up states are identical where finite."""
    size, n = 32768, 8
    edge = size // n  # first row of slab 1
    with fhn.Simulator(size, size) as sim:
        sim.init(2, 42)
        u, v = sim.download()
    u = u.reshape(size, size)
    u[edge - 1, 12345] = np.float32(9.28730297088623)   # last row of slab 0
    u[edge, 20000] = np.float32(7.935965061187744)      # first row of slab 1
    u = u.reshape(-1)
    with fhn.Simulator(size, size) as sim:
        sim.upload(u, v)
        want = int(sim.advance(40)[0])
        pu, pv = sim.download()
    assert want > 0
    with Ring(size, size, [0] * n, ghost=4) as ring:
        ring.upload(u, v)
        del u, v
        got = int(ring.advance(40)[0])
        ru, rv = ring.download()
    assert got == want
    fu, fv = np.isfinite(pu), np.isfinite(pv)
    assert np.array_equal(fu, np.isfinite(ru)) and np.array_equal(fv, np.isfinite(rv))
    assert np.array_equal(bits(ru)[fu], bits(pu)[fu]) and np.array_equal(bits(rv)[fv], bits(pv)[fv])


def test_engine_run_with_devices_backend():
    """engine.run / run_timed with Backend(devices=[...]): the reference's
    criterion-1 KAT (test_output.txt:8) and blow-up iteration
    (test_engine.cpp:95) on row slabs."""
    cfg = fhn.RunConfig(init_mode=1, nn=256, nm=256, iter_max=1000, nssp=1, seed=42,
                        backend=fhn.make_backend("cuda", devices=[0, 0, 0]))
    out = fhn.run(cfg, fhn.Gene(), fhn.init_center_square(256, 256, 42))
    assert fhn.checksum_hex(fhn.checksum(out.final_state)) == "1026befcb693b1e5"
    bufs = fhn.StepBuffers(fhn.init_center_square(16, 16, 42), fhn.make_backend("cuda", devices=[0, 0]))
    with pytest.raises(fhn.BlowUpError) as e:
        fhn.run_timed(bufs, fhn.Gene(dt=100), bufs.backend, 1000)
    assert e.value.iteration == 4


@pytest.mark.parametrize("driver", ["ring2", "ring1", "slabstepper"])
def test_blowup_replay_from_an_older_checkpoint(orc, driver):
    """A lattice that blows up late (iteration 3032 of a near-unstable gene,
    found with the oracle) advanced in calls of 100 iterations: the
    checkpoint is refreshed only every 2048 iterations, so the exact replay
    restarts from a state up to 2000 iterations before the failing call and
    must still report the oracle's iteration (engine.hpp:79)."""
    g7 = [0.2468, -0.3, 1.3, -0.1, 1.0, 0.06, 1.0]
    u0, v0 = orc.init(2, 32, 48, 11)
    ou, ov, obad = orc.run(32, 48, u0, v0, 4000, g7)
    assert obad == 3032
    if driver == "slabstepper":
        from paper_2102_10340_b200.slab import SlabStepper
        h = SlabStepper(32, 48, rank=0, world=1, ghost=4, device=0, transport="p2p")
        h.set_params(gene7(g7))
        h.upload(u0, v0)
        h.fill_ghosts()
        adv = h.advance
    else:
        h = Ring(32, 48, [0, 0] if driver == "ring2" else [0], ghost=4)
        h.set_params(gene7(g7))
        h.upload(u0, v0)
        adv = lambda k: int(h.advance(k)[0])  # noqa: E731
    done, bad = 0, 0
    while not bad:
        bad = adv(100)
        if not bad:
            done += 100
    u, v = h.download()
    h.close()
    assert done + bad == obad
    fu, fv = np.isfinite(ou), np.isfinite(ov)
    assert np.array_equal(fu, np.isfinite(u)) and np.array_equal(fv, np.isfinite(v))
    assert np.array_equal(bits(u)[fu], bits(ou)[fu]) and np.array_equal(bits(v)[fv], bits(ov)[fv])
