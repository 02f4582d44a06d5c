"""Parameter-plane sweeps on one batched device handle (reference
proj/include/rdcnn/sweep.hpp:16-350, minus the PNG panel rendering, which
is out of scope).

The reference runs |x|*|y| independent ``run()`` calls (optionally OpenMP
over cells, sweep.hpp:293-295) and post-processes every snapshot on the
host.  Here every cell is one grid of a batched handle (per-grid genes,
per-grid blow-up iteration), the snapshots stay on the device, and the
classifier statistics (min/max, nth_element median, active counts) are
computed there; only the per-grid scalars and the final states come back.
The labels and the CSV are bit-for-bit what the reference produces on the
same inputs (tests/test_sweep_gpu.py).
"""
from __future__ import annotations

import copy
import dataclasses
import math
import threading
from typing import List, Optional, Tuple

import numpy as np

from .engine import (DTYPES, Gene, RunConfig, ScheduleError, Simulator, gene_valid, init_center_square,
                     init_from_image, init_full_random, validate_config)

REGIMES = ("Homogeneous", "Patterned", "Growing", "BlowUp")
GENE_FIELDS = {"a": "a", "b": "b", "eps": "eps", "c": "c", "du": "Du", "dv": "Dv", "dt": "dt", "ka": "ka"}


def format_double(x: float) -> str:
    """std::to_chars(double) shortest round-trip form (config.hpp:103-107):
    the shortest of fixed and scientific notation, fixed on a tie."""
    if x == 0:
        return "-0" if math.copysign(1.0, x) < 0 else "0"
    if math.isinf(x):
        return "-inf" if x < 0 else "inf"
    if math.isnan(x):
        return "nan"
    r = repr(float(x))
    sign = "-" if r.startswith("-") else ""
    r = r.lstrip("-")
    mant, _, exp = r.partition("e")
    e = int(exp) if exp else 0
    ip, _, fp = mant.partition(".")
    digits = (ip + fp).lstrip("0")
    # decimal exponent of the first significant digit
    point = len(ip) + e  # position of the decimal point relative to ip+fp start
    lead_zeros = len(ip + fp) - len((ip + fp).lstrip("0"))
    point -= lead_zeros
    digits = digits.rstrip("0") or "0"
    n = len(digits)
    # fixed
    if point <= 0:
        fixed = "0." + "0" * (-point) + digits
    elif point >= n:
        # an integer: to_chars prints its exact decimal value in fixed form
        fixed = str(int(abs(float(x))))
    else:
        fixed = digits[:point] + "." + digits[point:]
    # scientific (printf %e style exponent: sign and at least two digits)
    se = point - 1
    sci = digits[0] + ("." + digits[1:] if n > 1 else "") + "e" + ("-" if se < 0 else "+") + f"{abs(se):02d}"
    return sign + (fixed if len(fixed) <= len(sci) else sci)


@dataclasses.dataclass
class ClassifierConfig:
    """sweep.hpp:31-37."""

    homogeneity_rel: float = 0.01
    homogeneity_floor: float = 0.01
    activity_rel: float = 0.1
    growth_factor: float = 10.0
    dip_tolerance: float = 0.10


@dataclasses.dataclass
class RegimeResult:
    label: str = "Patterned"
    final_range: float = 0.0
    final_active_fraction: float = 0.0
    activity_counts: List[int] = dataclasses.field(default_factory=list)


@dataclasses.dataclass
class SweepSpec:
    """sweep.hpp:118-131."""

    x_param: str
    x_values: List[float]
    y_param: str
    y_values: List[float]
    base_gene: Gene = dataclasses.field(default_factory=Gene)
    base_config: RunConfig = dataclasses.field(default_factory=RunConfig)
    keep_buffers: bool = False
    per_cell_seed: bool = False
    parallel_cells: bool = False  # accepted for API parity; cells always run batched
    fixed_range: Optional[Tuple[float, float]] = None
    classifier: ClassifierConfig = dataclasses.field(default_factory=ClassifierConfig)


@dataclasses.dataclass
class SweepCell:
    x_value: float = 0.0
    y_value: float = 0.0
    gene: Gene = dataclasses.field(default_factory=Gene)
    blew_up: bool = False
    blowup_iteration: int = 0
    outcome: RegimeResult = dataclasses.field(default_factory=RegimeResult)
    digest: int = 0
    final_u: Optional[np.ndarray] = None
    buffer: Optional[List[np.ndarray]] = None  # u frames when keep_buffers


@dataclasses.dataclass
class SweepResult:
    x_values: List[float]
    y_values: List[float]
    x_param: str
    y_param: str
    rows: int
    cols: int
    cells: List[SweepCell]
    labels_csv: str = ""
    panel: None = None  # PNG panel rendering is out of scope

    def at(self, yi: int, xi: int) -> SweepCell:
        return self.cells[yi * len(self.x_values) + xi]


def validate_sweep_spec(spec: SweepSpec):
    """sweep.hpp:133-142."""
    for p in (spec.x_param, spec.y_param):
        if p not in GENE_FIELDS:
            raise ValueError(f"unknown sweep parameter: {p}")
    if spec.x_param == spec.y_param:
        raise ValueError(f"sweep axes must differ (both are {spec.x_param})")
    if not spec.x_values or not spec.y_values:
        raise ValueError("sweep value lists must be non-empty")


def classify(frame_mins, frame_maxs, counts, cells: int, cc: ClassifierConfig, final_range: float) -> RegimeResult:
    """classify_outcome (sweep.hpp:77-112) from per-frame statistics."""
    res = RegimeResult()
    res.final_range = final_range
    gmin = min(float(frame_mins[-1]), *[float(m) for m in frame_mins])
    gmax = max(float(frame_maxs[-1]), *[float(m) for m in frame_maxs])
    global_range = gmax - gmin
    homog = max(cc.homogeneity_floor, cc.homogeneity_rel * global_range)
    res.activity_counts = [int(c) for c in counts]
    res.final_active_fraction = float(res.activity_counts[-1]) / float(cells)
    if res.final_range < homog:
        res.label = "Homogeneous"
        return res
    rising = True
    for k in range(len(res.activity_counts) - 1):
        rising &= float(res.activity_counts[k + 1]) >= (1.0 - cc.dip_tolerance) * float(res.activity_counts[k])
    grew = res.activity_counts[-1] >= max(1, int(cc.growth_factor * float(res.activity_counts[0])))
    res.label = "Growing" if (rising and grew) else "Patterned"
    return res


def classify_batch(frame_mins, frame_maxs, counts, cells: int, cc: ClassifierConfig, final_range):
    """classify() for every cell of a batch at once: arrays [frames, cells]
    (and final_range [cells]) in, per-cell labels and final active fractions
    out -- the same double-precision comparisons as classify(), elementwise
    (tests/test_sweep_host.py checks them against it).  Cells must be finite
    (blown-up cells are labelled before classification)."""
    mins = np.asarray(frame_mins, np.float64)
    maxs = np.asarray(frame_maxs, np.float64)
    cnt = np.asarray(counts, np.int64)
    fr = np.asarray(final_range, np.float64)
    global_range = maxs.max(axis=0) - mins.min(axis=0)
    homog = np.maximum(cc.homogeneity_floor, cc.homogeneity_rel * global_range)
    c = cnt.astype(np.float64)
    rising = np.all(c[1:] >= (1.0 - cc.dip_tolerance) * c[:-1], axis=0)
    grew = cnt[-1] >= np.maximum(1, (cc.growth_factor * c[0]).astype(np.int64))
    labels = np.where(fr < homog, "Homogeneous", np.where(rising & grew, "Growing", "Patterned"))
    return labels, c[-1] / float(cells)


def labels_csv(res: SweepResult) -> str:
    """sweep.hpp:227-247."""
    out = ["x_value,y_value,label,final_range,final_active_fraction,checksum\n"]
    xs = [format_double(x) for x in res.x_values]  # each axis value formatted once
    ys = [format_double(y) for y in res.y_values]
    for yi in range(len(res.y_values)):
        for xi in range(len(res.x_values)):
            c = res.at(yi, xi)
            line = f"{xs[xi]},{ys[yi]},{c.outcome.label},"
            if c.blew_up:
                out.append(line + ",,\n")
                continue
            out.append(line + "%.6g,%.6g,%016x\n" % (c.outcome.final_range, c.outcome.final_active_fraction,
                                                      c.digest))
    return "".join(out)


# Batched handles kept between sweeps of the same shape (like a caching
# allocator): creating and destroying a 4096 x 128^2 handle with its snapshot
# frames allocates and frees ~2.5 GiB of device memory per sweep, and the
# driver's release work made destruction cost 0.04-1.9 s.
_handles: dict = {}
_handles_lock = threading.Lock()
_MAX_CACHED = 8


def _take_handle(key) -> Simulator:
    with _handles_lock:
        sim = _handles.pop(key, None)
    if sim is None:
        rows, cols, batch, device, levels, prec, mode = key
        sim = Simulator(rows, cols, batch=batch, device=device, levels=levels, precision=prec, mode=mode)
    return sim


def _give_back(key, sim: Simulator) -> None:
    with _handles_lock:
        old = _handles.pop(key, None)
        _handles[key] = sim
        while len(_handles) > _MAX_CACHED:
            _handles.pop(next(iter(_handles))).close()
    if old is not None:
        old.close()


def release_cached_handles() -> None:
    """Free the device memory of the batched handles kept between sweeps."""
    with _handles_lock:
        sims = list(_handles.values())
        _handles.clear()
    for s in sims:
        s.close()


def _run_cells(cells: List[SweepCell], idx0: int, spec: SweepSpec, base: RunConfig,
               image: Optional[np.ndarray], device: int, levels: int, initial=None) -> None:
    """Runs `cells` (global indices idx0..) as one batched handle on `device`
    and fills in their outcomes (sweep.hpp:296-326)."""
    B, rows, cols = len(cells), base.nn, base.nm
    if B == 0:
        return
    prec = base.precision
    # base_config.backend.mode: strict (bit-exact, default) or the opt-in fast
    # arithmetic (validated statistically, tools/fast_mode_validation.py).
    key = (rows, cols, B, device, levels, prec, base.backend.mode)
    sim = _take_handle(key)
    sim.set_params([c.gene for c in cells])
    # initial states (init.hpp:67-82); the shared-seed default runs on the device
    sweeps_ka = "ka" in (spec.x_param, spec.y_param)
    if initial is not None:  # caller-supplied states, cells idx0.. of a (cells, rows*cols) pair
        u0, v0 = initial
        sim.upload(u0[idx0:idx0 + B], v0[idx0:idx0 + B])
    elif base.init_mode in (1, 2) and not spec.per_cell_seed:
        sim.init(base.init_mode, base.seed)
    elif base.init_mode == 3 and not sweeps_ka:
        sim.init_image(image, spec.base_gene.ka)
    else:
        U = np.empty((B, rows * cols), DTYPES[prec])
        V = np.empty_like(U)
        for idx, c in enumerate(cells):
            seed = base.seed + idx0 + idx if spec.per_cell_seed else base.seed
            if base.init_mode == 1:
                s = init_center_square(rows, cols, seed, prec)
            elif base.init_mode == 2:
                s = init_full_random(rows, cols, seed, prec)
            else:
                s = init_from_image(image, c.gene, prec)
            U[idx], V[idx] = s.u, s.v
        sim.upload(U, V)

    test_mod = base.iter_max // base.nssp
    F = base.nssp + 1
    sim.frames_reserve(F)
    sim.frame_capture(0)
    done = 0
    for f in range(1, F):
        bad = sim.advance(test_mod)
        for idx in np.nonzero(bad)[0]:
            c = cells[idx]
            if not c.blew_up:
                c.blew_up, c.blowup_iteration = True, done + int(bad[idx])
                c.outcome.label = "BlowUp"
        done += test_mod
        sim.frame_capture(f)

    stats = [sim.frame_stats(f) for f in range(F)]  # (mins, maxs, medians) per frame
    mins = np.stack([s[0] for s in stats])  # [F, B]
    maxs = np.stack([s[1] for s in stats])
    meds = np.stack([s[2] for s in stats])
    final_range = maxs[-1] - mins[-1]
    thr = spec.classifier.activity_rel * final_range
    counts = np.stack([sim.frame_active(f, meds[f], thr) for f in range(F)])  # [F, B]
    digests = sim.checksums()  # per grid, on the device
    # The cells keep their final u plane (sweep.hpp:318): the last snapshot
    # slot holds exactly it, so only u comes back, and each cell gets a view.
    frames_u = [sim.frame_download(f).reshape(B, -1) for f in range(F)] if spec.keep_buffers else None
    fu = frames_u[-1] if frames_u is not None else sim.frame_download(F - 1).reshape(B, -1)
    labels, fractions = classify_batch(mins, maxs, counts, rows * cols, spec.classifier, final_range)
    counts_t = counts.T.tolist()
    for idx, c in enumerate(cells):
        if c.blew_up:
            continue
        c.outcome = RegimeResult(label=str(labels[idx]), final_range=float(final_range[idx]),
                                 final_active_fraction=float(fractions[idx]), activity_counts=counts_t[idx])
        c.digest = int(digests[idx])
        c.final_u = fu[idx]
        if frames_u is not None:
            c.buffer = [fr[idx] for fr in frames_u]
    _give_back(key, sim)


def sweep_grid(spec: SweepSpec, image: Optional[np.ndarray] = None, device: int = 0,
               levels: int = 4, devices: Optional[List[int]] = None, initial=None) -> SweepResult:
    """sweep_grid (sweep.hpp:255-326) as one batched device run, or with
    `devices`, the cells split in contiguous chunks over several GPUs.

    ``initial``: optional (u, v) host arrays of shape (cells, rows*cols), the
    cells' initial states in sweep order (y outer, x inner), uploaded instead
    of drawing them from the seed (e.g. to sweep from an evolved state)."""
    validate_sweep_spec(spec)
    base = dataclasses.replace(spec.base_config)
    issues = validate_config(base, spec.base_gene)
    if base.init_mode == 3 and image is not None:
        issues = [i for i in issues if not i.startswith("MissingImage")]
    if issues:
        raise ValueError(issues[0].split(": ", 1)[-1])
    if base.iter_max % base.nssp != 0:
        raise ScheduleError("nssp must divide iter_max for sweep cells")
    if base.init_mode == 3:
        if image is None:
            raise ValueError("typ=3 requires an image")
        base.nn, base.nm = int(image.shape[0]), int(image.shape[1])
    cells: List[SweepCell] = []
    fx, fy = GENE_FIELDS[spec.x_param], GENE_FIELDS[spec.y_param]
    # gene_valid is a conjunction of per-field tests, so with two distinct
    # swept fields every cell is valid iff every x and every y value is (with
    # the base gene's other fields); otherwise the cell loop below finds and
    # reports the first invalid cell in sweep order.
    bg = spec.base_gene
    separable_ok = (fx != fy and
                    all(gene_valid(dataclasses.replace(bg, **{fx: float(x)})) for x in spec.x_values) and
                    all(gene_valid(dataclasses.replace(bg, **{fy: float(y)})) for y in spec.y_values))
    for y in spec.y_values:
        for x in spec.x_values:
            if separable_ok:
                g = copy.copy(bg)
                setattr(g, fx, float(x))
                setattr(g, fy, float(y))
            else:
                g = dataclasses.replace(bg, **{fx: float(x), fy: float(y)})
                if not gene_valid(g):
                    raise ValueError(f"sweep cell gene invalid at {spec.x_param}={format_double(x)} "
                                     f"{spec.y_param}={format_double(y)}")
            cells.append(SweepCell(x_value=float(x), y_value=float(y), gene=g))

    if initial is not None:
        n = len(spec.x_values) * len(spec.y_values)
        u0, v0 = (np.asarray(a).reshape(n, -1) for a in initial)
        if u0.shape[1] != base.nn * base.nm or v0.shape != u0.shape:
            raise ValueError(f"initial states must be ({n}, {base.nn * base.nm}) arrays")
        initial = (u0, v0)
    devs = list(devices) if devices else [device]
    bounds = np.linspace(0, len(cells), len(devs) + 1).astype(int)
    jobs = [(cells[lo:hi], int(lo), dev) for lo, hi, dev in zip(bounds[:-1], bounds[1:], devs) if hi > lo]
    if len(jobs) == 1:
        _run_cells(jobs[0][0], jobs[0][1], spec, base, image, jobs[0][2], levels, initial)
    elif jobs:
        # Replicas only: independent cells, no exchange; the C-ABI
        # calls release the GIL, so the devices advance concurrently.
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(len(jobs)) as ex:
            list(ex.map(lambda j: _run_cells(j[0], j[1], spec, base, image, j[2], levels, initial), jobs))
    rows, cols = base.nn, base.nm
    res = SweepResult(list(spec.x_values), list(spec.y_values), spec.x_param, spec.y_param, rows, cols, cells)
    res.labels_csv = labels_csv(res)
    return res
