"""Host-side sweep post-processing: the batched classifier equals the
per-cell one (classify_outcome, sweep.hpp:77-112) on random and boundary
statistics.  CPU only."""
import numpy as np

from paper_2102_10340_b200.sweep import ClassifierConfig, classify, classify_batch


def _check(mins, maxs, counts, cells, cc, final_range):
    labels, fractions = classify_batch(mins, maxs, counts, cells, cc, final_range)
    for i in range(mins.shape[1]):
        r = classify(mins[:, i], maxs[:, i], counts[:, i], cells, cc, float(final_range[i]))
        assert labels[i] == r.label, i
        assert fractions[i] == r.final_active_fraction, i


def test_classify_batch_random():
    rng = np.random.default_rng(3)
    F, B, cells = 6, 2000, 128 * 128
    cc = ClassifierConfig()
    mins = rng.normal(-1.0, 0.5, (F, B))
    maxs = mins + rng.exponential(1.0, (F, B)) * (rng.random((F, B)) < 0.7)
    counts = np.cumsum(rng.integers(-50, 400, (F, B)), axis=0).clip(0, cells)
    final_range = maxs[-1] - mins[-1]
    _check(mins, maxs, counts, cells, cc, final_range)


def test_classify_batch_boundaries():
    cc = ClassifierConfig()
    F, cells = 3, 1000
    cols = []
    # final range exactly at the homogeneity threshold (floor and relative), a
    # dip exactly at the tolerance, growth exactly at the factor, zero counts
    for fr, gr in ((cc.homogeneity_floor, 0.0), (cc.homogeneity_rel * 10.0, 10.0), (1.0, 1.0)):
        for c in ([0, 0, 0], [10, 10 * (1 - cc.dip_tolerance), 100], [10, 20, int(cc.growth_factor * 10)],
                  [10, 20, int(cc.growth_factor * 10) - 1], [100, 50, 900], [1, 1, 1]):
            cols.append((fr, gr, c))
    mins = np.array([[0.0] * len(cols)] * F)
    maxs = np.array([[gr for _, gr, _ in cols]] * F)
    counts = np.array([c for _, _, c in cols], np.float64).T.round().astype(np.int64)
    final_range = np.array([fr for fr, _, _ in cols])
    _check(mins, maxs, counts, cells, cc, final_range)


def test_invalid_sweep_cell_reported_in_sweep_order():
    """sweep.hpp: the first invalid cell (y outer, x inner) is named; the
    separable fast path must not change which one."""
    import pytest

    from paper_2102_10340_b200.engine import RunConfig
    from paper_2102_10340_b200.sweep import SweepSpec, sweep_grid

    cfg = RunConfig()
    cfg.nn = cfg.nm = 16
    cfg.iter_max = 10
    cfg.nssp = 1
    spec = SweepSpec("du", [0.1, -0.2, 0.3], "dv", [0.5, -1.0], base_config=cfg)
    with pytest.raises(ValueError, match=r"du=-0.2 dv=0.5"):
        sweep_grid(spec)
    spec = SweepSpec("du", [0.1, 0.2], "dv", [0.5, -1.0], base_config=cfg)
    with pytest.raises(ValueError, match=r"du=0.1 dv=-1"):
        sweep_grid(spec)
