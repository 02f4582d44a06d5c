"""Python mirror of the reference's time-stepping API, on the CUDA backend.

Same names, argument meaning and error behaviour as the reference C++ API
(paths relative to /root/reference/proj/include/rdcnn/):

=====================  ====================================================
this module            reference
=====================  ====================================================
Gene                   gene.hpp:13-24 (defaults), gene_valid :34-36
GridState              grid.hpp:31-53 (rows=NN, cols=NM, planes u, v)
Backend/make_backend   backend.hpp:12-50 (+ the ``cuda`` kind)
StepBuffers            kernels.hpp:22-38 (state lives on the device)
step                   kernels.hpp:233-259 (swap always, False on non-finite)
run / RunOutput        engine.hpp:54-94 (snapshots every iter_max/nssp)
run_timed              engine.hpp:98-106 (bare loop, BlowUpError(iter))
BlowUpError            engine.hpp:20-26
ScheduleError          engine.hpp:15-17
init_*                 init.hpp:20-82
checksum               grid.hpp:101-116
=====================  ====================================================

Everything computes through the C-ABI (include/rdcnn_cuda.h).  The CPU
backends of the reference (reference/blocked/parallel/shift) are not part of
this framework: asking for one raises ``ValueError`` instead of silently
running something else.
"""
from __future__ import annotations

import ctypes
import dataclasses
import time
from typing import Callable, List, Optional

import numpy as np

from ._lib import RDCNN_FAST, RDCNN_STRICT, ParamsF32, ParamsF64, check, load

DTYPES = {"single": np.float32, "double": np.float64}

__all__ = [
    "Gene", "GridState", "Backend", "make_backend", "StepBuffers", "step", "run",
    "run_timed", "RunConfig", "RunOutput", "SnapshotBuffer", "BlowUpError",
    "ScheduleError", "init_center_square", "init_full_random", "init_from_image",
    "initial_state", "checksum", "checksum_hex", "Simulator", "gene_valid",
    "params_from_gene", "validate_config",
]


# ---------------------------------------------------------------------------
# Domain types
# ---------------------------------------------------------------------------

@dataclasses.dataclass
class Gene:
    """Parameter set of one RD-CNN instance (gene.hpp:13-24)."""

    a: float = -0.3
    b: float = 1.3
    eps: float = -0.1
    c: float = 1.0
    Du: float = 0.06
    Dv: float = 1.0
    dt: float = 0.1
    ka: float = 1.0

    def to_vector(self) -> List[float]:
        """Kernel order [dt, a, b, eps, c, Du, Dv] (gene.hpp:39-41)."""
        return [self.dt, self.a, self.b, self.eps, self.c, self.Du, self.Dv]


def gene_valid(g: Gene) -> bool:
    """All fields finite and dt, Du, Dv >= 0 (gene.hpp:27-36)."""
    vals = [g.a, g.b, g.eps, g.c, g.Du, g.Dv, g.dt, g.ka]
    return all(np.isfinite(vals)) and g.dt >= 0 and g.Du >= 0 and g.Dv >= 0


def params_from_gene(g: Gene, precision: str = "single"):
    """make_params<T> (model.hpp:24-32): narrowed to fp32 by the C-ABI, or fp64 as is."""
    if precision == "double":
        return ParamsF64(*[float(x) for x in g.to_vector()])
    lib = load()
    arr = (ctypes.c_double * 7)(*g.to_vector())
    out = ParamsF32()
    lib.rdcnn_params_from_gene(arr, ctypes.byref(out))
    return out


def gene_batch(genes, precision: str = "single"):
    """Batches (sweeps): the kernel-order vectors of many genes narrowed in
    one numpy pass, round-to-nearest like make_params<float>
    (model.hpp:24-32), as a ctypes array of ParamsF32 (ParamsF64 for
    double) sharing the numpy buffer -- what rdcnn_sim_set_params takes."""
    kind = ParamsF64 if precision == "double" else ParamsF32
    vec = np.array([g.to_vector() for g in genes], np.float64)
    arr = np.ascontiguousarray(vec if precision == "double" else vec.astype(np.float32))
    out = (kind * len(genes)).from_buffer(arr)
    out._keep = arr  # the ctypes view must keep its buffer alive
    return out


class GridState:
    """The paired u/v layers of a rows x cols toroidal lattice (grid.hpp:31-53)."""

    def __init__(self, rows: int, cols: int, u=None, v=None, dtype=None):
        if rows < 3 or cols < 3:
            raise ValueError("grid must be at least 3x3")
        self.rows, self.cols = int(rows), int(cols)
        n = self.rows * self.cols
        if dtype is None:
            dtype = u.dtype if isinstance(u, np.ndarray) and u.dtype == np.float64 else np.float32
        self.dtype = np.dtype(dtype)
        self.u = np.zeros(n, dtype) if u is None else np.ascontiguousarray(u, dtype).reshape(n)
        self.v = np.zeros(n, dtype) if v is None else np.ascontiguousarray(v, dtype).reshape(n)

    @property
    def precision(self) -> str:
        return "double" if self.dtype == np.float64 else "single"

    def cells(self) -> int:
        return self.rows * self.cols

    def copy(self) -> "GridState":
        return GridState(self.rows, self.cols, self.u.copy(), self.v.copy(), self.dtype)

    def __eq__(self, other) -> bool:  # bitwise, like the defaulted operator==
        if not (isinstance(other, GridState) and self.rows == other.rows and self.cols == other.cols
                and self.dtype == other.dtype):
            return False
        it = np.uint32 if self.dtype == np.float32 else np.uint64
        return (np.array_equal(self.u.view(it), other.u.view(it))
                and np.array_equal(self.v.view(it), other.v.view(it)))


class BlowUpError(RuntimeError):
    """First iteration whose result holds a non-finite entry (engine.hpp:20-26)."""

    def __init__(self, iteration: int):
        super().__init__(f"blow-up: non-finite state after iteration {iteration}")
        self.iteration = int(iteration)


class ScheduleError(RuntimeError):
    """nssp does not divide iter_max (engine.hpp:15-17, :59-61)."""


BACKEND_KINDS = ("cuda",)
_CPU_KINDS = ("reference", "shift", "blocked", "parallel")


@dataclasses.dataclass
class Backend:
    """Backend selection (backend.hpp:14-21); this framework provides ``cuda``.

    ``mode`` is ``"strict"`` (bit-exact with the reference exact-order
    backends) or ``"fast"`` (FMA-contracted, tolerance-checked).  ``levels``
    caps the time levels fused per launch (1, 2, 4, 8).
    """

    kind: str = "cuda"
    tile_rows: int = 64
    tile_cols: int = 64
    threads: int = 0
    mode: str = "strict"
    device: int = 0
    levels: int = 4
    # Two or more entries: row slabs of the lattice on these devices (the
    # in-process fused peer ring, slab.Ring; fp32).  The multi-GPU
    # counterpart of the reference's row-band parallelism (kernels.hpp:153-174).
    devices: Optional[List[int]] = None

    def exact_order(self) -> bool:
        return self.mode == "strict"


def make_backend(name: str = "cuda", tile_rows: int = 64, tile_cols: int = 64, threads: int = 0,
                 mode: str = "strict", device: int = 0, levels: int = 4,
                 devices: Optional[List[int]] = None) -> Backend:
    """backend.hpp:44-50 plus the ``cuda`` kind; unknown names raise ValueError."""
    if tile_rows < 1 or tile_cols < 1:
        raise ValueError("tile dimensions must be >= 1")
    if threads < 0:
        raise ValueError("thread count must be >= 0")
    if name in _CPU_KINDS:
        raise ValueError(f"backend '{name}' is a reference CPU backend; this framework provides "
                         "'cuda' only (see INTEGRATION.md for running both side by side)")
    if name not in BACKEND_KINDS:
        raise ValueError(f"unknown backend: {name} (expected cuda)")
    if mode not in ("strict", "fast"):
        raise ValueError(f"unknown mode: {mode} (expected strict|fast)")
    if levels not in (1, 2, 4, 8):
        raise ValueError("levels must be 1, 2, 4 or 8")
    return Backend(name, tile_rows, tile_cols, threads, mode, device, levels,
                   list(devices) if devices else None)


# ---------------------------------------------------------------------------
# Device handle
# ---------------------------------------------------------------------------

def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class Simulator:
    """Owner of one device state (C-ABI handle): batch x rows x cols, two planes."""

    def __init__(self, rows: int, cols: int, batch: int = 1, device: int = 0, mode: str = "strict",
                 levels: int = 4, seg_rows: int = 0, precision: str = "single", persistent: int = 0):
        """``persistent``: the one-launch cluster path for small single fp32
        lattices (rdcnn_sim_set_persistent): 0 automatic, 1 required, -1 off."""
        self._lib = load()
        self.rows, self.cols, self.batch, self.device = int(rows), int(cols), int(batch), int(device)
        self.mode = mode
        if precision not in DTYPES:
            raise ValueError(f"unknown precision {precision} (expected single|double)")
        self.precision = precision
        self.dtype = np.dtype(DTYPES[precision])
        self._f64 = precision == "double"
        h = ctypes.c_void_p()
        m = RDCNN_FAST if mode == "fast" else RDCNN_STRICT
        if mode not in ("strict", "fast"):
            raise ValueError(f"unknown mode {mode}")
        if self._f64:
            check(self._lib.rdcnn_sim_create_f64(self.rows, self.cols, self.batch, self.device, ctypes.byref(h)))
            levels = min(levels, 4)
        else:
            check(self._lib.rdcnn_sim_create(self.rows, self.cols, self.batch, self.device, m, ctypes.byref(h)))
        self._h = h
        self.set_tuning(levels, seg_rows)
        check(self._lib.rdcnn_sim_set_persistent(self._h, int(persistent)))
        L = self._lib
        self._up = L.rdcnn_sim_upload_f64 if self._f64 else L.rdcnn_sim_upload
        self._down = L.rdcnn_sim_download_f64 if self._f64 else L.rdcnn_sim_download

    # lifetime
    def close(self):
        if getattr(self, "_h", None):
            self._lib.rdcnn_sim_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # configuration
    def set_tuning(self, levels: int = 4, seg_rows: int = 0):
        check(self._lib.rdcnn_sim_set_tuning(self._h, int(levels), int(seg_rows)))
        self.levels = int(levels)

    def set_params(self, genes):
        kind = ParamsF64 if self._f64 else ParamsF32
        genes = [genes] if isinstance(genes, (Gene, ParamsF32, ParamsF64)) else list(genes)
        fn = self._lib.rdcnn_sim_set_params_f64 if self._f64 else self._lib.rdcnn_sim_set_params
        if len(genes) > 1 and all(isinstance(g, Gene) for g in genes):
            arr = gene_batch(genes, self.precision)
            check(fn(self._h, arr, len(genes)))
            return
        arr = (kind * len(genes))()
        for k, g in enumerate(genes):
            arr[k] = g if isinstance(g, kind) else params_from_gene(g, self.precision)
        check(fn(self._h, arr, len(genes)))

    # state transfer
    def _shape_n(self) -> int:
        return self.batch * self.rows * self.cols

    def upload(self, u: np.ndarray, v: np.ndarray):
        u = np.ascontiguousarray(u, self.dtype)
        v = np.ascontiguousarray(v, self.dtype)
        if u.size != self._shape_n() or v.size != self._shape_n():
            raise ValueError("upload size does not match batch*rows*cols")
        check(self._up(self._h, _ptr(u), _ptr(v)))

    def upload_ptr(self, u_ptr: int, v_ptr: int):
        check(self._up(self._h, ctypes.c_void_p(u_ptr), ctypes.c_void_p(v_ptr)))

    def download(self, u: Optional[np.ndarray] = None, v: Optional[np.ndarray] = None):
        n = self._shape_n()
        u = np.empty(n, self.dtype) if u is None else u
        v = np.empty(n, self.dtype) if v is None else v
        check(self._down(self._h, _ptr(u), _ptr(v)))
        return u, v

    def download_ptr(self, u_ptr: int, v_ptr: int):
        check(self._down(self._h, ctypes.c_void_p(u_ptr), ctypes.c_void_p(v_ptr)))

    def init(self, typ: int, seed: int):
        check(self._lib.rdcnn_sim_init(self._h, int(typ), ctypes.c_uint64(seed)))

    def init_image(self, px: np.ndarray, ka: float = 1.0):
        px = np.ascontiguousarray(px, np.uint8)
        if px.size != self.rows * self.cols:
            raise ValueError("image size does not match rows*cols")
        check(self._lib.rdcnn_sim_init_image(self._h, _ptr(px), float(ka)))

    # stepping
    def advance(self, steps: int) -> np.ndarray:
        """Advance every grid; returns first_bad[batch] (0 = stayed finite)."""
        bad = (ctypes.c_long * self.batch)()
        check(self._lib.rdcnn_sim_advance(self._h, int(steps), bad))
        return np.array(bad[:], dtype=np.int64)

    def checksums(self) -> np.ndarray:
        """checksum (grid.hpp:100-126) of every grid, computed on the device."""
        out = np.empty(self.batch, np.uint64)
        check(self._lib.rdcnn_sim_checksums(self._h, out.ctypes.data))
        return out

    def elapsed_ms(self) -> float:
        ms = ctypes.c_double()
        check(self._lib.rdcnn_sim_elapsed_ms(self._h, ctypes.byref(ms)))
        return ms.value

    def launch_count(self) -> int:
        n = ctypes.c_long()
        check(self._lib.rdcnn_sim_launch_count(self._h, ctypes.byref(n)))
        return n.value

    def stream(self) -> int:
        s = ctypes.c_void_p()
        check(self._lib.rdcnn_sim_stream(self._h, ctypes.byref(s)))
        return s.value or 0

    # snapshot store (device-resident frames for batched analysis)
    def frames_reserve(self, nframes: int):
        check(self._lib.rdcnn_sim_frames_reserve(self._h, int(nframes)))

    def frame_capture(self, slot: int):
        check(self._lib.rdcnn_sim_frame_capture(self._h, int(slot)))

    def frame_download(self, slot: int) -> np.ndarray:
        u = np.empty(self._shape_n(), self.dtype)
        check(self._lib.rdcnn_sim_frame_download(self._h, int(slot), _ptr(u)))
        return u

    def frame_stats(self, slot: int):
        """Per grid: (min, max, median) of the u plane in `slot` (nth_element(n/2))."""
        mn, mx, med = (np.empty(self.batch, np.float64) for _ in range(3))
        check(self._lib.rdcnn_sim_frame_stats(self._h, int(slot), _ptr(mn), _ptr(mx), _ptr(med)))
        return mn, mx, med

    def frame_active(self, slot: int, medians: np.ndarray, thresholds: np.ndarray) -> np.ndarray:
        med = np.ascontiguousarray(medians, np.float64)
        thr = np.ascontiguousarray(thresholds, np.float64)
        out = np.empty(self.batch, np.int64)
        check(self._lib.rdcnn_sim_frame_active(self._h, int(slot), _ptr(med), _ptr(thr), _ptr(out)))
        return out

    def frame_normalize(self, slot: int, grid: int, lo: float, hi: float) -> np.ndarray:
        """normalize_frame(_fixed) on the device; slot < 0 = the current state."""
        out = np.empty(self.rows * self.cols, np.uint8)
        check(self._lib.rdcnn_sim_frame_normalize(self._h, int(slot), int(grid), float(lo), float(hi),
                                                  _ptr(out)))
        return out.reshape(self.rows, self.cols)

    def frame_normalize_auto(self, slot: int = -1, grid: int = 0):
        """normalize_frame (frame.hpp:28-44) on the device with the plane's own
        min/max; returns (rows x cols uint8 image, lo, hi).  slot < 0 = the
        current state."""
        out = np.empty(self.rows * self.cols, np.uint8)
        lo, hi = ctypes.c_double(), ctypes.c_double()
        check(self._lib.rdcnn_sim_frame_normalize_auto(self._h, int(slot), int(grid), _ptr(out), ctypes.byref(lo),
                                                       ctypes.byref(hi)))
        return out.reshape(self.rows, self.cols), lo.value, hi.value

    def frame_normalize_auto_ptr(self, out_ptr: int, slot: int = -1, grid: int = 0):
        """As frame_normalize_auto into caller memory (rows*cols bytes)."""
        lo, hi = ctypes.c_double(), ctypes.c_double()
        check(self._lib.rdcnn_sim_frame_normalize_auto(self._h, int(slot), int(grid), ctypes.c_void_p(out_ptr),
                                                       ctypes.byref(lo), ctypes.byref(hi)))
        return lo.value, hi.value

    def init_image_ptr(self, px_ptr: int, ka: float = 1.0):
        """init_image from caller memory (rows*cols uint8 pixels, e.g. pinned)."""
        check(self._lib.rdcnn_sim_init_image(self._h, ctypes.c_void_p(px_ptr), float(ka)))

    def device_state(self):
        u, v = ctypes.c_void_p(), ctypes.c_void_p()
        check(self._lib.rdcnn_sim_device_state(self._h, ctypes.byref(u), ctypes.byref(v)))
        return u.value, v.value


class Pipeline:
    """A stream of independent lattices of one shape (images to process,
    initial states to evolve) through ``depth`` device handles, one host
    thread each.  Lattice i runs on handle i % depth as upload -> advance ->
    download, so its host<->device copies overlap another lattice's advance:
    the C-ABI calls release the GIL and every handle has its own stream.
    Results are those of one Simulator running the jobs one after another.

    ``sims``: existing (e.g. warmed) Simulators of that shape to use as the
    first handles; the rest are created with ``kw`` (Simulator arguments)."""

    def __init__(self, rows: int, cols: int, depth: int = 2, sims: Optional[List[Simulator]] = None, **kw):
        if depth < 1:
            raise ValueError("depth must be >= 1")
        self.sims = list(sims or [])[:depth]
        for s in self.sims:
            if (s.rows, s.cols, s.batch) != (rows, cols, 1):
                raise ValueError("pipeline simulators must be single rows x cols lattices")
        self._owned = [Simulator(rows, cols, **kw) for _ in range(depth - len(self.sims))]
        self.sims += self._owned

    def set_params(self, gene):
        for s in self.sims:
            s.set_params(gene)

    def run(self, jobs, steps: int) -> np.ndarray:
        """``jobs``: (u_in, v_in, u_out, v_out) host pointers per lattice
        (pinned memory for full copy bandwidth; an output pair must not be
        shared by jobs on different handles).  Advances each lattice ``steps``
        iterations; returns its first bad iteration (0 = stayed finite), the
        output holding the state after ``steps`` either way (engine.hpp:79)."""
        from concurrent.futures import ThreadPoolExecutor

        jobs = list(jobs)
        bad = np.zeros(len(jobs), np.int64)
        d = len(self.sims)
        # Per job: the advance's device time (CUDA events on its handle), so
        # callers can split end-to-end time into device and copy time.
        self.last_device_ms = np.zeros(len(jobs), np.float64)

        def lane(k: int):
            sim = self.sims[k]
            for i in range(k, len(jobs), d):
                u_in, v_in, u_out, v_out = jobs[i]
                sim.upload_ptr(u_in, v_in)
                bad[i] = sim.advance(steps)[0]
                self.last_device_ms[i] = sim.elapsed_ms()
                sim.download_ptr(u_out, v_out)

        if d == 1:
            lane(0)
        else:
            with ThreadPoolExecutor(d) as ex:
                for f in [ex.submit(lane, k) for k in range(min(d, len(jobs)))]:
                    f.result()
        return bad

    def run_images(self, jobs, steps: int, ka: float = 1.0) -> np.ndarray:
        """Edge detection over a stream of images (the reference's typ=3 run,
        init.hpp:58 + frame.hpp:28-44): per job (pixels_ptr, out_ptr), both
        rows*cols bytes of host memory -- init_image, ``steps`` iterations,
        the final u plane normalised on the device into ``out``.  Returns
        each job's first bad iteration (0 = stayed finite)."""
        from concurrent.futures import ThreadPoolExecutor

        jobs = list(jobs)
        bad = np.zeros(len(jobs), np.int64)
        d = len(self.sims)
        self.last_device_ms = np.zeros(len(jobs), np.float64)

        def lane(k: int):
            sim = self.sims[k]
            for i in range(k, len(jobs), d):
                px, out = jobs[i]
                sim.init_image_ptr(px, ka)
                bad[i] = sim.advance(steps)[0]
                self.last_device_ms[i] = sim.elapsed_ms()
                sim.frame_normalize_auto_ptr(out)

        if d == 1:
            lane(0)
        else:
            with ThreadPoolExecutor(d) as ex:
                for f in [ex.submit(lane, k) for k in range(min(d, len(jobs)))]:
                    f.result()
        return bad

    def close(self):
        for s in self._owned:
            s.close()
        self._owned = []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


# ---------------------------------------------------------------------------
# Reference-shaped API
# ---------------------------------------------------------------------------

class StepBuffers:
    """Double buffer of one lattice (kernels.hpp:22-38).

    The state lives on the device; ``front`` downloads it on access, so a
    loop of ``step`` calls never round-trips through the host.
    """

    def __init__(self, initial: GridState, backend: Optional[Backend] = None):
        be = backend or Backend()
        self.backend = be
        if be.devices and len(be.devices) > 1:
            if initial.precision != "single":
                raise ValueError("multi-device row slabs run fp32 lattices only")
            from .slab import Ring
            self.sim = Ring(initial.rows, initial.cols, be.devices, ghost=be.levels, mode=be.mode)
        else:
            self.sim = Simulator(initial.rows, initial.cols, 1, be.device, be.mode, be.levels,
                                 precision=initial.precision)
        self.sim.upload(initial.u, initial.v)
        self._rows, self._cols = initial.rows, initial.cols
        self._gene_key = None

    def rows(self) -> int:
        return self._rows

    def cols(self) -> int:
        return self._cols

    @property
    def front(self) -> GridState:
        u, v = self.sim.download()
        return GridState(self._rows, self._cols, u, v, self.sim.dtype)

    def set_front(self, state: GridState):
        self.sim.upload(state.u, state.v)

    def _use_gene(self, gene: Gene):
        key = tuple(gene.to_vector())
        if key != self._gene_key:
            self.sim.set_params(gene)
            self._gene_key = key


def _require_cuda(backend: Optional[Backend]) -> Backend:
    be = backend or Backend()
    if be.kind != "cuda":
        raise ValueError(f"backend '{be.kind}' is not provided by this framework")
    return be


def step(bufs: StepBuffers, gene: Gene, backend: Optional[Backend] = None) -> bool:
    """One iteration; False when any new value is non-finite (swap still happens)."""
    _require_cuda(backend)
    bufs._use_gene(gene)
    bad = bufs.sim.advance(1)
    return int(bad[0]) == 0


def run_timed(bufs: StepBuffers, gene: Gene, backend: Optional[Backend], iters: int) -> float:
    """engine.hpp:98-106: bare loop; returns device seconds; BlowUpError(iter)."""
    _require_cuda(backend)
    bufs._use_gene(gene)
    bad = bufs.sim.advance(int(iters))
    if bad[0]:
        raise BlowUpError(int(bad[0]))
    return bufs.sim.elapsed_ms() / 1e3


@dataclasses.dataclass
class RunConfig:
    """config.hpp:30-41 (typ 1 = CenterSquare, 2 = FullRandom, 3 = Image)."""

    init_mode: int = 1
    nn: int = 512
    nm: int = 512
    image_path: Optional[str] = None
    image_size: Optional[int] = None
    iter_max: int = 10000
    nssp: int = 5
    seed: int = 1
    backend: Backend = dataclasses.field(default_factory=Backend)
    precision: str = "single"


def validate_config(cfg: RunConfig, gene: Gene) -> List[str]:
    """All invariant violations as messages (config.hpp:62-95); empty = runnable."""
    issues = []
    if cfg.nn < 3 or cfg.nm < 3:
        issues.append(f"InvalidSize: grid must be at least 3x3, got {cfg.nn}x{cfg.nm}")
    if cfg.init_mode == 1 and (cfg.nn < 11 or cfg.nm < 11):
        issues.append(f"InvalidSize: typ=1 needs room for the 11x11 seed square, got {cfg.nn}x{cfg.nm}")
    if cfg.iter_max < 1:
        issues.append(f"InvalidSchedule: iter_max must be >= 1, got {cfg.iter_max}")
    if cfg.nssp < 1 or cfg.nssp > cfg.iter_max:
        issues.append(f"InvalidSchedule: nssp must satisfy 1 <= nssp <= iter_max, got nssp={cfg.nssp} "
                      f"iter_max={cfg.iter_max}")
    elif cfg.iter_max >= 1 and cfg.iter_max % cfg.nssp != 0:
        issues.append(f"InvalidSchedule: nssp ({cfg.nssp}) must divide iter_max ({cfg.iter_max})")
    if cfg.init_mode == 3 and not cfg.image_path:
        issues.append("MissingImage: typ=3 requires an image path")
    vals = [gene.a, gene.b, gene.eps, gene.c, gene.Du, gene.Dv, gene.dt, gene.ka]
    if not all(np.isfinite(vals)):
        issues.append("NonFiniteGene: gene has non-finite fields")
    elif not gene_valid(gene):
        issues.append("NonFiniteGene: gene invariant violated (need dt >= 0, Du >= 0, Dv >= 0)")
    return issues


@dataclasses.dataclass
class SnapshotBuffer:
    rows: int = 0
    cols: int = 0
    frames_u: List[np.ndarray] = dataclasses.field(default_factory=list)
    frames_v: List[np.ndarray] = dataclasses.field(default_factory=list)
    labels: List[int] = dataclasses.field(default_factory=list)

    def frame_count(self) -> int:
        return len(self.labels)


@dataclasses.dataclass
class RunOutput:
    final_state: Optional[GridState] = None
    snapshots: SnapshotBuffer = dataclasses.field(default_factory=SnapshotBuffer)
    wall_seconds: float = 0.0
    snapshot_elapsed: List[float] = dataclasses.field(default_factory=list)


def run(cfg: RunConfig, gene: Gene, initial: GridState,
        on_snapshot: Optional[Callable[[int, float], None]] = None) -> RunOutput:
    """engine.hpp:54-94 on the device: state stays resident between snapshots."""
    if cfg.precision not in DTYPES:
        raise ValueError(f"unknown precision: {cfg.precision}")
    if (cfg.precision == "double") != (initial.dtype == np.float64):
        raise ValueError(f"initial state dtype {initial.dtype} does not match precision={cfg.precision}")
    if initial.rows != cfg.nn or initial.cols != cfg.nm:
        raise ValueError("initial state shape does not match config")
    if cfg.nssp < 1 or cfg.nssp > cfg.iter_max or cfg.iter_max % cfg.nssp != 0:
        raise ScheduleError(f"nssp ({cfg.nssp}) must divide iter_max ({cfg.iter_max})")
    be = _require_cuda(cfg.backend)
    test_mod = cfg.iter_max // cfg.nssp
    out = RunOutput()
    snaps = out.snapshots
    snaps.rows, snaps.cols = cfg.nn, cfg.nm
    snaps.frames_u.append(initial.u.copy())
    snaps.frames_v.append(initial.v.copy())
    snaps.labels.append(0)
    bufs = StepBuffers(initial, be)
    bufs._use_gene(gene)
    t0 = time.perf_counter()
    done = 0
    while done < cfg.iter_max:
        bad = bufs.sim.advance(test_mod)
        if bad[0]:
            raise BlowUpError(done + int(bad[0]))
        done += test_mod
        elapsed = time.perf_counter() - t0
        u, v = bufs.sim.download()
        snaps.frames_u.append(u)
        snaps.frames_v.append(v)
        snaps.labels.append(done)
        out.snapshot_elapsed.append(elapsed)
        if on_snapshot:
            on_snapshot(done, elapsed)
    out.wall_seconds = time.perf_counter() - t0
    out.final_state = GridState(cfg.nn, cfg.nm, snaps.frames_u[-1].copy(), snaps.frames_v[-1].copy(),
                                initial.dtype)
    return out


# ---------------------------------------------------------------------------
# Initial states and digest
# ---------------------------------------------------------------------------

def init_center_square(rows: int, cols: int, seed: int, precision: str = "single") -> GridState:
    """typ=1 (init.hpp:34-48), init_center_square<float|double>."""
    if rows < 11 or cols < 11:
        raise ValueError(f"typ=1 needs a grid of at least 11x11, got {rows}x{cols}")
    s = GridState(rows, cols, dtype=DTYPES[precision])
    L = load()
    fn = L.rdcnn_init_center_square_host_f64 if precision == "double" else L.rdcnn_init_center_square_host
    check(fn(rows, cols, ctypes.c_uint64(seed), _ptr(s.u), _ptr(s.v)))
    return s


def init_full_random(rows: int, cols: int, seed: int, precision: str = "single") -> GridState:
    """typ=2 (init.hpp:23-30), init_full_random<float|double>."""
    s = GridState(rows, cols, dtype=DTYPES[precision])
    L = load()
    fn = L.rdcnn_init_full_random_host_f64 if precision == "double" else L.rdcnn_init_full_random_host
    check(fn(rows, cols, ctypes.c_uint64(seed), _ptr(s.u), _ptr(s.v)))
    return s


def init_from_image(px: np.ndarray, gene: Gene, precision: str = "single") -> GridState:
    """typ=3 (init.hpp:51-64): u = v = T(ka) * T(px/255.0)."""
    px = np.asarray(px, np.uint8)
    if px.ndim != 2 or px.shape[0] < 3 or px.shape[1] < 3:
        raise ValueError("image must be at least 3x3")
    t = DTYPES[precision]
    x = t(gene.ka) * (px.astype(np.float64) / 255.0).astype(t)
    return GridState(px.shape[0], px.shape[1], x.reshape(-1), x.reshape(-1).copy(), t)


def initial_state(cfg: RunConfig, gene: Gene, image: Optional[np.ndarray] = None) -> GridState:
    if cfg.init_mode == 1:
        return init_center_square(cfg.nn, cfg.nm, cfg.seed, cfg.precision)
    if cfg.init_mode == 2:
        return init_full_random(cfg.nn, cfg.nm, cfg.seed, cfg.precision)
    if cfg.init_mode == 3:
        if image is None:
            raise ValueError("typ=3 requires an image")
        return init_from_image(image, gene, cfg.precision)
    raise ValueError("typ must be 1, 2 or 3")


def checksum(state: GridState) -> int:
    """FNV-1a 64 over u then v raw bytes (grid.hpp:101-116)."""
    L = load()
    fn = L.rdcnn_checksum_f64 if state.dtype == np.float64 else L.rdcnn_checksum_f32
    return int(fn(_ptr(state.u), _ptr(state.v), state.cells()))


def checksum_hex(x: int) -> str:
    return f"{x:016x}"
