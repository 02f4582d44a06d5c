"""Batched parameter sweeps (§8f2) and frame normalisation (§8f4) on the
device, against the reference's own sweep_grid labels CSV (golden) and the
reference formulas (sweep.hpp:48-112, frame.hpp:28-66)."""
import json
import os

import numpy as np
import pytest

import paper_2102_10340_b200 as fhn
from paper_2102_10340_b200.sweep import ClassifierConfig, SweepSpec, format_double, sweep_grid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def golden_sweeps():
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)["sweeps"]


def spec_from(d):
    cfg = fhn.RunConfig(init_mode=d.get("typ", 1), nn=d["nn"], nm=d["nm"], iter_max=d["iter_max"],
                        nssp=d["nssp"], seed=d.get("seed", 42))
    return SweepSpec(x_param=d["x_param"], x_values=d["xs"], y_param=d["y_param"], y_values=d["ys"],
                     base_config=cfg, per_cell_seed=d.get("per_cell_seed", False))


# --- CPU: host logic -----------------------------------------------------------

def test_format_double_matches_to_chars_examples():
    assert [format_double(x) for x in (0.0, 1.0, 0.02, 0.3, 5.0, -0.05, 1e-5, 1e21, 0.0001, 123456.0)] == \
        ["0", "1", "0.02", "0.3", "5", "-0.05", "1e-05", "1e+21", "1e-04", "123456"]
    try:
        from oracle.oracle import Reference
        ref = Reference()
    except (OSError, FileNotFoundError):
        return
    rng = np.random.default_rng(1)
    vals = list(10.0 ** rng.uniform(-40, 40, 2000)) + list(rng.uniform(-1e3, 1e3, 500))
    assert [format_double(x) for x in vals] == [ref.format_double(x) for x in vals]


def test_sweep_spec_validation():
    from paper_2102_10340_b200.sweep import validate_sweep_spec
    with pytest.raises(ValueError, match="unknown sweep parameter"):
        validate_sweep_spec(SweepSpec("zz", [1], "dv", [1]))
    with pytest.raises(ValueError, match="must differ"):
        validate_sweep_spec(SweepSpec("du", [1], "du", [1]))
    with pytest.raises(ValueError, match="non-empty"):
        validate_sweep_spec(SweepSpec("du", [], "dv", [1]))


def test_classifier_on_synthetic_counts():
    """classify_outcome branches (sweep.hpp:77-112) on hand-built statistics."""
    from paper_2102_10340_b200.sweep import classify
    cc = ClassifierConfig()
    # homogeneous: final range below max(0.01, 0.01 * global range)
    r = classify([0.0, 0.5], [1.0, 0.5], [3, 0], 100, cc, 0.0)
    assert r.label == "Homogeneous"
    # growing: counts rise (with a tolerated 5% dip) and grow 10x
    r = classify([0.0] * 4, [1.0] * 4, [10, 50, 48, 120], 1000, cc, 1.0)
    assert r.label == "Growing" and r.final_active_fraction == 0.12
    # a 20% dip breaks "rising"
    assert classify([0.0] * 4, [1.0] * 4, [10, 50, 40, 120], 1000, cc, 1.0).label == "Patterned"


# --- GPU ---------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("case", golden_sweeps(), ids=lambda c: f"{c['spec']['x_param']}x{c['spec']['y_param']}"
                         f"_{c['spec']['nn']}")
def test_sweep_labels_equal_reference(case):
    res = sweep_grid(spec_from(case["spec"]))
    assert res.labels_csv == case["labels_csv"]


@pytest.mark.gpu
def test_frame_stats_and_normalisation(oracle):
    rows, cols, B = 48, 64, 3
    genes = [fhn.Gene(Du=0.06), fhn.Gene(Du=0.3), fhn.Gene(a=-0.05)]
    with fhn.Simulator(rows, cols, batch=B) as sim:
        sim.set_params(genes)
        sim.init(2, 5)
        sim.frames_reserve(2)
        sim.frame_capture(0)
        sim.advance(50)
        sim.frame_capture(1)
        U = sim.frame_download(1).reshape(B, -1)
        mn, mx, med = sim.frame_stats(1)
        thr = np.array([0.05, 0.1, 0.2])
        cnt = sim.frame_active(1, med, thr)
        for g in range(B):
            x = U[g]
            assert mn[g] == float(x.min()) and mx[g] == float(x.max())
            assert med[g] == float(np.partition(x, x.size // 2)[x.size // 2])  # nth_element(n/2)
            assert cnt[g] == int((np.abs(x.astype(np.float64) - med[g]) > thr[g]).sum())
            img = sim.frame_normalize(1, g, mn[g], mx[g])
            scale = 255.0 / (mx[g] - mn[g])
            y = (x.astype(np.float64) - mn[g]) * scale
            want = np.clip(np.floor(y + 0.5), 0, 255).astype(np.uint8)  # lround for y >= 0
            assert np.array_equal(img.reshape(-1), want)
            assert (sim.frame_normalize(1, g, 1.0, 1.0) == 128).all()
    # the current state (slot -1) equals the last capture
    with fhn.Simulator(rows, cols) as sim:
        sim.init(1, 42)
        sim.advance(10)
        u, _ = sim.download()
        a = sim.frame_normalize(-1, 0, float(u.min()), float(u.max()))
        assert a.shape == (rows, cols)


@pytest.mark.gpu
@pytest.mark.parametrize("per_cell_seed", (False, True))
def test_sweep_split_over_devices_identical(per_cell_seed):
    """cfg4 as 'replicas only': the cells split over several
    handles/devices (here three handles on GPU 0, advanced concurrently from
    threads) give the same labels CSV, digests and blow-ups as one batch."""
    from paper_2102_10340_b200.engine import RunConfig
    from paper_2102_10340_b200.sweep import SweepSpec, sweep_grid

    cfg = RunConfig()
    cfg.nn = cfg.nm = 64
    cfg.iter_max, cfg.nssp, cfg.init_mode = 400, 4, 2
    spec = SweepSpec("du", list(np.linspace(0.02, 0.9, 7)), "dt", [0.1, 0.5, 40.0], base_config=cfg,
                     per_cell_seed=per_cell_seed)
    one = sweep_grid(spec)
    split = sweep_grid(spec, devices=[0, 0, 0])
    assert split.labels_csv == one.labels_csv
    assert [c.digest for c in split.cells] == [c.digest for c in one.cells]
    assert [c.blowup_iteration for c in split.cells] == [c.blowup_iteration for c in one.cells]
    assert any(c.blew_up for c in one.cells)


@pytest.mark.gpu
def test_sweep_from_supplied_initial_states():
    """sweep_grid(initial=(u, v)): uploading exactly the states the seed would
    draw gives the reference's labels CSV byte for byte; other states change it."""
    case = golden_sweeps()[0]
    spec = spec_from(case["spec"])
    d = case["spec"]
    n = len(d["xs"]) * len(d["ys"])
    st = fhn.init_center_square(d["nn"], d["nm"], d.get("seed", 42))
    u = np.tile(st.u, (n, 1))
    v = np.tile(st.v, (n, 1))
    assert sweep_grid(spec, initial=(u, v)).labels_csv == case["labels_csv"]
    u2 = u.copy()
    u2[:, :] = fhn.init_full_random(d["nn"], d["nm"], 5).u
    assert sweep_grid(spec, initial=(u2, v)).labels_csv != case["labels_csv"]
    with pytest.raises(ValueError):
        sweep_grid(spec, initial=(u[:, :-1], v[:, :-1]))


@pytest.mark.gpu
def test_sweep_handle_reuse():
    """Consecutive sweeps of one shape reuse the cached batched handle; the
    result does not depend on it (golden labels both times, then after a
    sweep of another spec on the same handle)."""
    from paper_2102_10340_b200 import sweep as sw
    sw.release_cached_handles()
    case = golden_sweeps()[0]
    spec = spec_from(case["spec"])
    assert sweep_grid(spec).labels_csv == case["labels_csv"]
    assert len(sw._handles) == 1
    h = next(iter(sw._handles.values()))
    other = spec_from(dict(case["spec"], xs=[0.05, 0.6]))
    sweep_grid(other)
    assert next(iter(sw._handles.values())) is h
    assert sweep_grid(spec).labels_csv == case["labels_csv"]
    sw.release_cached_handles()
    assert not sw._handles
