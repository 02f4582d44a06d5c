#!/usr/bin/env python
"""Benchmark of the FitzHugh-Nagumo RD-CNN time-stepping path on B200.

Workload (BASELINE.json configs[1], "cfg2"): 4096 x 4096 fp32 torus,
typ=1 seed 42, slow-growth gene (a = -0.05), strict (bit-exact) arithmetic.
One bench "step" = one advance of --iters-per-step iterations (default 10000,
so the default 10 timed steps are exactly the 100k-iteration cfg2 run).

Metric: Mcell-updates/s = rows*cols*iterations / seconds / 1e6
(reference bench.hpp:29-33).  The state (2 planes x 2 buffers = 256 MiB) is
larger than the 126 MB L2, so no explicit L2 flush is needed.

  python bench.py                         # N=1, our sm_100a path
  python bench.py --impl reference        # the reference CPU path (oracle/_ref)
  torchrun --nproc-per-node N bench.py --gpus N   # row slabs, fused peer halo exchange
  torchrun --nproc-per-node N bench.py --gpus N --workload cfg5   # one 32768^2 torus over N GPUs

For N > 1 each rank owns a 4096-row slab of a (4096*N) x 4096 torus (weak
scaling, cfg2) or 32768/N rows of one 32768^2 torus (strong scaling, cfg5,
BASELINE configs[4]) and exchanges `levels` halo rows with its ring
neighbours per block.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GENE7 = [0.1, -0.05, 1.3, -0.1, 1.0, 0.06, 1.0]  # dt,a,b,eps,c,Du,Dv: slow growth
DEFAULT_GENE7 = [0.1, -0.3, 1.3, -0.1, 1.0, 0.06, 1.0]  # gene.hpp:13-24
BYTES_PER_CELL_UPDATE = 16  # read u,v + write u,v, fp32
FLOPS_PER_CELL_UPDATE = 27  # 26 add/sub/mul + 1 divide


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", default="cfg2", choices=("cfg2", "cfg5", "cfg1", "cfg3", "cfg4"),
                    help="cfg2 (default): a size x size torus per GPU, weak scaling; cfg5: ONE "
                         "size x size torus (default 32768) split over the N GPUs, strong scaling; "
                         "cfg1 (256^2 x 1000) / cfg3 (8192^2 image x 200): one lattice per GPU, "
                         "independent replicas; cfg4: the 64 x 64 (Du, Dv) sweep of 128^2 x 5000 "
                         "lattices, one plane per GPU")
    ap.add_argument("--size", type=int, default=None,
                    help="cfg2: rows = cols per GPU (default 4096); cfg5: the lattice edge (32768)")
    ap.add_argument("--iters-per-step", type=int, default=None,
                    help="default 10000 (cfg2), 100 (cfg5)")
    ap.add_argument("--levels", type=int, default=4, choices=(1, 2, 4, 8))
    ap.add_argument("--seg-rows", type=int, default=0)
    ap.add_argument("--mode", default="strict", choices=("strict", "fast"))
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="lattices through the e2e pipeline (0: the workload's default)")
    ap.add_argument("--e2e-states", action="store_true",
                    help="cfg3: time the float state stream (upload u,v -> advance -> download u,v) instead of "
                         "the image stream (pixels -> advance -> normalised edge map)")
    ap.add_argument("--e2e-depth", type=int, default=0,
                    help="lattices in flight in the e2e pipeline (0: the workload's default; 1: one after another)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="budget of the cpu_baseline sample on rank 0")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--slab", action="store_true",
                    help="run the multi-GPU slab path even at N=1 (a world-1 ring)")
    ap.add_argument("--devices", default=None,
                    help="single-process multi-GPU run (no torchrun): comma-separated CUDA ordinals, one "
                         "row slab each, e.g. 0,1,2,3 (default for --gpus N without torchrun: 0..N-1); "
                         "repeating an ordinal puts several slabs on one GPU (functional tests only)")
    ap.add_argument("--ring", action="store_true",
                    help="run the slab workloads through the in-process ring (rdcnn_ring_*) even at N=1")
    ap.add_argument("--transport", default="auto", choices=("auto", "p2p", "nccl"),
                    help="slab halo exchange: fused peer stores in the step kernel (p2p), NCCL, "
                         "or auto (p2p unless a rank cannot map its neighbours' memory)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------

class Workload:
    """BASELINE.json configs the bench runs.

    cfg2: init_center_square(size, size, 42), slow-growth gene a=-0.05; at N>1
          each GPU owns a size-row slab of a (size*N) x size torus (weak scaling).
    cfg5: init_full_random(size, size, 42) with the reference default gene, ONE
          size x size torus (default 32768^2) row-slabbed over the N GPUs (strong
          scaling)."""

    def __init__(self, args, world: int):
        self.name = args.workload
        self.replicas = self.name in ("cfg1", "cfg3", "cfg4")
        self.batch = 1  # grids per GPU (cfg4: the sweep's cells)
        if self.name == "cfg4":
            n = args.size or 128
            self.cols = self.rows_rank = self.rows_global = n
            self.batch = 64 * 64
            self.typ, self.gene7 = 1, DEFAULT_GENE7
            self.iters = args.iters_per_step or 5000
            self.e2e_steps, self.e2e_depth = 2, 1
            self.scaling = "weak"
            self.desc = (f"cfg4: FHN RD-CNN sweep of {self.batch} {n}x{n} fp32 tori per GPU, typ=1 seed 42, "
                         "Du = linspace(0.02,0.70,64) x Dv = linspace(0.50,1.20,64) on the reference default "
                         f"gene, {self.iters} iterations per step"
                         + ("; independent planes, one per GPU" if world > 1 else ""))
        elif self.replicas:
            n = args.size or (256 if self.name == "cfg1" else 8192)
            self.cols = self.rows_rank = self.rows_global = n
            self.typ, self.gene7 = (1 if self.name == "cfg1" else 3), DEFAULT_GENE7
            self.iters = args.iters_per_step or (1000 if self.name == "cfg1" else 200)
            self.e2e_steps = 20 if self.name == "cfg1" else 12
            # cfg3 is edge detection over a stream of independent images:
            # three in flight, so one's upload and another's download overlap
            # a third's advance (depth 2/3/4: 637k/798k/805k).  Every other
            # workload is one evolving lattice whose steps depend on each
            # other, so its e2e runs them strictly one after another.
            self.e2e_depth = 3 if self.name == "cfg3" else 1
            self.scaling = "weak"
            self.desc = (f"{self.name}: FHN RD-CNN {n}x{n} fp32 torus per GPU, "
                         + ("typ=1 seed 42" if self.typ == 1 else "typ=3 synthetic 8-bit image (SURVEY §8d)")
                         + f", reference default gene, {self.iters} iterations per step"
                         + ("; independent replicas, one per GPU" if world > 1 else ""))
        elif self.name == "cfg5":
            self.cols = args.size or 32768
            self.rows_global = self.cols
            if self.rows_global % world:
                raise SystemExit(f"cfg5: {self.rows_global} rows do not split over {world} GPUs")
            self.rows_rank = self.rows_global // world
            self.typ, self.gene7 = 2, DEFAULT_GENE7
            self.iters = args.iters_per_step or 100
            self.e2e_steps = 2
            self.e2e_depth = 1
            self.scaling = "strong"
            self.desc = (f"cfg5: FHN RD-CNN {self.rows_global}x{self.cols} fp32 torus, typ=2 (full "
                         f"random) seed 42, reference default gene, {self.iters} iterations per step")
        else:
            n = args.size or 4096
            self.cols = n
            self.rows_rank = n
            self.rows_global = n * world
            self.typ, self.gene7 = 1, GENE7
            self.iters = args.iters_per_step or 10000
            self.e2e_steps = 3
            self.e2e_depth = 1
            self.scaling = "weak"
            self.desc = (f"cfg2: FHN RD-CNN {n}x{n} fp32 torus per GPU, typ=1 seed 42, "
                         f"slow-growth gene a=-0.05, {self.iters} iterations per step")

    def published(self):
        """the paper's fastest published implementation of this
        step (PyCUDA on a Tesla P100, 10 000 iterations, Mcells/s) at this
        lattice edge, or None when it publishes none at this size."""
        table = {256: 1941.0, 512: 7581.0, 1024: 13059.0, 2048: 14198.0, 4096: 14545.0}
        if self.name in ("cfg2", "cfg1") and self.cols in table and self.rows_rank == self.cols:
            return table[self.cols], (f"PyCUDA {self.cols}^2 x 10000 iterations on a Tesla P100-PCIE, "
                                      f"{table[self.cols]:.0f} Mcells/s (BASELINE.md §1, PAPER.md:271-274)")
        return None, None

    def axes(self):
        """cfg4's sweep axes: Du along x, Dv along y."""
        import numpy as np
        return list(np.linspace(0.02, 0.70, 64)), list(np.linspace(0.50, 1.20, 64))

    def gene(self, fhn):
        g = self.gene7
        base = fhn.Gene(dt=g[0], a=g[1], b=g[2], eps=g[3], c=g[4], Du=g[5], Dv=g[6])
        if self.name != "cfg4":
            return base
        import dataclasses
        xs, ys = self.axes()
        return [dataclasses.replace(base, Du=float(x), Dv=float(y)) for y in ys for x in xs]

    def pixels(self):
        """cfg3 image: SURVEY §8d pattern (checker blocks 37x53 + a sine ramp), 8-bit."""
        import numpy as np
        n = self.cols
        i = np.arange(n)[:, None]
        j = np.arange(n)[None, :]
        x = np.where(((i // 37) + (j // 53)) % 2 == 1, 0.8, 0.2) + 0.1 * np.sin(0.05 * i)
        return np.clip(np.round(x * 255), 0, 255).astype(np.uint8)

    def ref_state(self, ref):
        """The initial state through the reference's own initialisers."""
        if self.typ != 3:
            return ref.init(self.typ, self.rows_global, self.cols, 42)
        from paper_2102_10340_b200 import imageio
        fd, path = tempfile.mkstemp(suffix=".pgm")
        os.close(fd)
        try:
            imageio.write_pgm(path, self.pixels())
            _, _, u, v = ref.init_image(path, 1.0)
        finally:
            os.unlink(path)
        return u, v

def config_dict(wl: "Workload", args, world: int, use_slab: bool, transport):
    """The line's ``config``: the workload both arms measure (the reference
    arm prints the same dict; its bounded sample is described in its
    cpu_baseline.sample)."""
    n = wl.cols
    per_rank_cells = wl.rows_rank * n * wl.batch
    return {
        "workload": (wl.desc
                     + (f"; global {wl.rows_global}x{n} row-slabbed ({wl.rows_rank} rows per "
                        f"GPU), halo exchange: "
                        + ("fused peer reads in the step kernel" if transport == "p2p"
                           else "NCCL send/recv overlapped with the interior kernel")
                        if use_slab else "")),
        "rows": wl.rows_global, "cols": n, "iterations_per_step": wl.iters, "levels_per_launch": args.levels,
        "mode": args.mode,
        "l2": (f"double-buffered state {2 * 8 * per_rank_cells / 2**20:.0f} MiB/GPU "
               + ("> 126 MB L2 (no flush needed)" if 2 * 8 * per_rank_cells > 126e6
                  else "fits in L2: a 256 MiB buffer is written before every step, each step "
                       "timed on its own")),
        **({"grids": wl.batch} if wl.batch > 1 else {}),
        "parallelism": (f"slab{world}" if use_slab else f"replicas{world}" if world > 1 else "single"),
        **({"transport": transport} if use_slab else {}),
    }


def predicted_layout(wl: "Workload", args, world: int):
    """(use_slab, transport) our arm will use for this workload."""
    use_slab = (world > 1 or args.slab or args.ring or bool(args.devices)) and not wl.replicas
    transport = ("p2p" if args.transport == "auto" else args.transport) if use_slab else None
    return use_slab, transport


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
              "enforced.power.limit")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        # nvidia-smi takes a few hundred ms to start: wait (before the timed
        # region opens) until it has written its first sample, so that short
        # regions (cfg1) are sampled too.
        t_end = time.time() + 3.0
        while self.proc is not None and time.time() < t_end and self.proc.poll() is None:
            if os.path.getsize(self.path) > 0:
                break
            time.sleep(0.02)
        with open(self.path) as f:
            self.skip = len(f.readlines())  # samples taken before the region: not counted
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, pw, lim, reasons = [], [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            lines = f.readlines()
        # The region's samples; a region shorter than the 100 ms period falls
        # back to the last sample before it (and says so).
        in_region = lines[getattr(self, "skip", 0):]
        pre_region = not in_region
        for line in in_region or lines[-1:]:
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx.append(float(p[2]))
            except ValueError:
                continue
            try:
                pw.append(float(p[3]))
                lim.append(float(p[9]))
            except (ValueError, IndexError):
                pass
            for name, val in zip(names, p[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm),
                "power_w": round(statistics.median(pw), 1) if pw else None,
                "power_limit_w": max(lim) if lim else None,
                **({"pre_region_sample": True} if pre_region and sm else {})}


def ncu_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(path):
        return None, None
    with open(path) as f:
        d = json.load(f)
    return d.get("dram_bytes_per_launch"), d.get("cell_updates_per_launch")


def host_threads() -> int:
    """Every host core this process may run on.  torchrun exports
    OMP_NUM_THREADS=1 to each rank, so the reference's OpenMP default would be
    one thread there; the reference arm passes this count explicitly to the
    reference's Backend instead (backend.hpp:44-50, threads > 0)."""
    try:
        return len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        return os.cpu_count() or 1


def ref_sweep_sample(wl: "Workload", ref, threads: int):
    """cfg4 on the reference: its own sweep_grid with parallel_cells (OpenMP
    over cells, sweep.hpp:293-295) on the first a x b cells of the plane, two
    cells per host thread, the full iteration count.  Returns (cell-updates/s
    in M, seconds, cells)."""
    ref.set_threads(threads)
    xs, ys = wl.axes()
    want = max(4, 2 * threads)
    a = min(len(xs), max(1, int(want ** 0.5)))
    b = min(len(ys), max(1, -(-want // a)))
    t0 = time.perf_counter()
    ref.sweep_labels("du", xs[:a], "dv", ys[:b], gene7=wl.gene7, nn=wl.rows_global, nm=wl.cols,
                     iter_max=wl.iters, nssp=5 if wl.iters % 5 == 0 else 1, seed=42, parallel_cells=True)
    sec = time.perf_counter() - t0
    return a * b * wl.rows_global * wl.cols * wl.iters / sec / 1e6, sec, a * b


def cpu_baseline_sample(wl: "Workload", budget_s: float):
    """The reference's own parallel backend (oracle/_ref, reference headers
    compiled read-only) on a bounded prefix of the same workload."""
    from oracle.oracle import Reference
    ref = Reference()
    threads = host_threads()
    if wl.name == "cfg4":
        value, sec, ncells = ref_sweep_sample(wl, ref, threads)
        return {"value": round(value, 2), "unit": "Mcell-updates/s", "cores": threads, "kind": "reference",
                "sample": f"reference sweep_grid (oracle/_ref, parallel_cells, {threads} OpenMP threads) on "
                          f"{ncells} cells of the plane, {wl.rows_global}x{wl.cols} x {wl.iters} iterations "
                          f"each, snapshots + classifier included ({sec:.2f} s)"}
    R, C = wl.rows_global, wl.cols
    u, v = wl.ref_state(ref)
    # calibrate with 2 iterations, then size the sample to the budget
    u, v, _, sec = ref.run_timed(R, C, u, v, 2, wl.gene7, backend="parallel", threads=threads)
    per_iter = max(sec / 2, 1e-6)
    iters = int(max(2, min(2000, budget_s / per_iter)))
    u, v, bad, sec = ref.run_timed(R, C, u, v, iters, wl.gene7, backend="parallel", threads=threads)
    value = R * C * iters / sec / 1e6
    return {"value": round(value, 2), "unit": "Mcell-updates/s", "cores": threads,
            "kind": "reference",
            "sample": f"reference parallel backend (oracle/_ref, {threads} OpenMP threads), "
                      f"{R}x{C} typ={wl.typ} seed 42 ({wl.name} gene), iterations 3..{iters + 2} "
                      f"({sec:.2f} s) of the same run"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def bench_reference_sweep(args, wl, ref, threads, world):
    """cfg4 reference arm: each step = the reference sweep_grid on a bounded
    sub-plane (two cells per host thread, full 128^2 x 5000 each)."""
    for _ in range(args.warmup):
        ref_sweep_sample(wl, ref, threads)
    total, work = 0.0, 0.0
    for _ in range(args.steps):
        value, sec, ncells = ref_sweep_sample(wl, ref, threads)
        total += sec
        work += value * sec
    value = work / total
    sample = (f"reference sweep_grid (oracle/_ref, parallel_cells) on {ncells} cells of the plane per step, "
              f"{wl.rows_global}x{wl.cols} x {wl.iters} iterations each, {threads} threads on {cpu_model()}")
    line = {
        "impl": "reference", "metric": "Mcell-updates/s", "value": round(value, 2),
        "unit": "Mcell-updates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": wl.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(wl, args, world, *predicted_layout(wl, args, world)),
        "cpu_baseline": {"value": round(value, 2), "unit": "Mcell-updates/s", "cores": threads,
                         "kind": "reference", "sample": sample, "cells_per_step_sampled": ncells},
        "e2e": {"value": round(value, 2), "unit": "Mcell-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def bench_reference(args, rank, world):
    if rank != 0:
        return
    from oracle.oracle import Reference
    wl = Workload(args, world)
    ref = Reference()
    R, C = wl.rows_global, wl.cols  # the same global lattice our arm advances
    threads = host_threads()
    if wl.name == "cfg4":
        bench_reference_sweep(args, wl, ref, threads, world)
        return
    u, v = wl.ref_state(ref)
    # size each step to ~2 s of CPU work so the whole run stays within minutes
    u, v, _, sec = ref.run_timed(R, C, u, v, 2, wl.gene7, backend="parallel", threads=threads)
    iters = int(max(1, min(wl.iters, 2.0 / max(sec / 2, 1e-6))))
    for _ in range(args.warmup):
        u, v, _, _ = ref.run_timed(R, C, u, v, iters, wl.gene7, backend="parallel", threads=threads)
    total = 0.0
    for _ in range(args.steps):
        u, v, bad, sec = ref.run_timed(R, C, u, v, iters, wl.gene7, backend="parallel", threads=threads)
        total += sec
    value = R * C * iters * args.steps / total / 1e6
    sample = (f"reference parallel backend via run_timed (oracle/_ref = reference headers), "
              f"{threads} threads on {cpu_model()}; each step = {iters} iterations of {R}x{C}")
    line = {
        "impl": "reference", "metric": "Mcell-updates/s", "value": round(value, 2),
        "unit": "Mcell-updates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": wl.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(wl, args, world, *predicted_layout(wl, args, world)),
        "cpu_baseline": {"value": round(value, 2), "unit": "Mcell-updates/s", "cores": threads,
                         "kind": "reference", "sample": sample, "iterations_per_step_sampled": iters,
                         "iterations_timed": f"{args.warmup * iters + 3}..{(args.warmup + args.steps) * iters + 2} "
                                             "of the run (1-based), after 2 calibration iterations and the "
                                             "warmup steps"},
        "e2e": {"value": round(value, 2), "unit": "Mcell-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def bench_ours(args, rank, world, local_rank, ring_devices=None):
    """Our arm.  ``ring_devices``: the single-process multi-GPU mode -- one
    process drives every slab through the in-process ring (rdcnn_ring_*, one
    host thread per device); world = len(ring_devices)."""
    import numpy as np
    import torch

    import paper_2102_10340_b200 as fhn

    # RDCNN_BENCH_ONE_DEVICE=1 (testing only): every rank on cuda:0 with a gloo
    # group, so the N>1 path (IPC peer ring, barriers, max over ranks) can be
    # exercised on a one-GPU box.  Never used for reported numbers.
    one_dev = os.environ.get("RDCNN_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    red_dev = "cpu" if one_dev else "cuda"
    wl = Workload(args, world)
    n = wl.cols
    S = wl.iters
    gene = wl.gene(fhn)
    dist = None
    ring = None
    if ring_devices is not None and wl.replicas:
        raise SystemExit(f"{wl.name} runs independent replicas: launch N > 1 under torch.distributed.run")
    if world > 1 and ring_devices is None:
        import torch.distributed as dist
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    launches = 0
    if ring_devices is not None:
        # One process, N row slabs (rdcnn_ring_*): every device's blocks are
        # enqueued by its own host thread; ring.elapsed_ms() is the max over
        # the devices' CUDA-event times of each advance.
        ring = fhn.Ring(wl.rows_global, n, ring_devices, ghost=args.levels, mode=args.mode)
        ring.set_params(gene)
        ring.init(wl.typ, 42)
        for _ in range(args.warmup):
            ring.advance(S)
        torch.cuda.synchronize()
        with ClockSampler(ring_devices[0]) as clocks:
            t_ms = 0.0
            for _ in range(args.steps):
                bad = ring.advance(S)
                t_ms += ring.elapsed_ms()
                launches += ring.launch_count()
                if bad.any():
                    raise RuntimeError(f"blow-up at iteration {int(bad[0])}")
        cells_global = wl.rows_global * n
    elif (world == 1 and not args.slab) or wl.replicas:
        sim = fhn.Simulator(wl.rows_global, n, batch=wl.batch, device=local_rank, mode=args.mode,
                            levels=args.levels, seg_rows=args.seg_rows)
        sim.set_params(gene)
        if wl.typ == 3:
            sim.init_image(wl.pixels(), 1.0)
        else:
            sim.init(wl.typ, 42)
        stream = torch.cuda.ExternalStream(sim.stream(), device=local_rank)
        for _ in range(args.warmup):
            sim.advance(S)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        # A state smaller than L2 (cfg1) would stay cached between steps: write
        # a 256 MiB buffer before every step, outside its own timed events.
        flush = (torch.empty(256 * 2**20, dtype=torch.uint8, device=f"cuda:{local_rank}")
                 if 2 * 8 * wl.rows_rank * n * wl.batch <= 126e6 else None)
        with ClockSampler(local_rank) as clocks:
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            t_ms = 0.0
            if flush is None:
                ev0.record(stream)
            for _ in range(args.steps):
                if flush is not None:
                    flush.zero_()
                    torch.cuda.synchronize()
                    ev0.record(stream)
                bad = sim.advance(S)
                if flush is not None:
                    ev1.record(stream)
                    torch.cuda.synchronize()
                    t_ms += ev0.elapsed_time(ev1)
                launches += sim.launch_count()
                if bad.any():
                    raise RuntimeError(f"blow-up at iteration {int(bad[bad > 0].min())}")
            if flush is None:
                ev1.record(stream)
                torch.cuda.synchronize()
                t_ms = ev0.elapsed_time(ev1)
        t = torch.tensor([t_ms], device=red_dev)
        if dist is not None:  # replicas: the job takes as long as its slowest GPU
            dist.barrier()
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())
        cells_global = wl.rows_global * n * wl.batch * (world if wl.replicas else 1)
    else:
        from paper_2102_10340_b200.slab import SlabStepper
        rows_global = wl.rows_global
        slab = SlabStepper(rows_global, n, rank, world, ghost=args.levels, device=local_rank,
                           mode=args.mode, seg_rows=args.seg_rows, transport=args.transport)
        slab.set_params(gene)
        slab.init(wl.typ, 42)
        slab.fill_ghosts()
        hs = ctypes.c_void_p()
        fhn.load().rdcnn_sim_stream(slab._h, ctypes.byref(hs))
        stream = torch.cuda.ExternalStream(hs.value, device=local_rank)  # the slab's compute stream
        for _ in range(args.warmup):
            slab.advance(S)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        with ClockSampler(local_rank) as clocks:
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            l0 = slab.launches
            ev0.record(stream)
            bad = 0
            for _ in range(args.steps):
                bad = bad or slab.advance(S)
            ev1.record(stream)
            torch.cuda.synchronize()
            launches = slab.launches - l0
        t = torch.tensor([ev0.elapsed_time(ev1)], device=red_dev)
        if dist is not None:
            dist.barrier()
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())
        cells_global = rows_global * n
        if bad:
            raise RuntimeError(f"blow-up in slab run near iteration {bad}")

    total_updates = cells_global * S * args.steps
    value = total_updates / (t_ms / 1e3) / 1e6
    clock_info = clocks.summary()

    # ---- roofline of the dominant kernel (the K-level wavefront stencil) ----
    peaks, peak_kind = measured_peaks()
    per_rank_cells = wl.rows_rank * n * wl.batch
    use_slab = (world > 1 or args.slab or ring is not None) and not wl.replicas
    transport = "p2p" if ring is not None else slab.transport if use_slab else None
    levels = args.levels
    # One K-level block = one launch per slab; slabs sharing a device (the
    # one-GPU functional ring) run their launches one after another.
    slabs_per_device = (max(ring_devices.count(d) for d in ring_devices) if ring is not None else 1)
    blocks_per_rank = max(S * args.steps // levels, 1) * slabs_per_device
    avg_launch_s = (t_ms / 1e3) / blocks_per_rank
    alg_bytes_per_launch = BYTES_PER_CELL_UPDATE * per_rank_cells * levels
    achieved_gbs = alg_bytes_per_launch / avg_launch_s / 1e9
    traffic, traffic_units = ncu_traffic()
    if traffic_units != per_rank_cells * levels:
        traffic = None  # the committed capture is of another launch size
    sm_mhz = clock_info.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    max_mhz = peaks.get("sm_max_mhz", 1965.0)
    fp32_peak_tops = 148 * 128 * sm_mhz * 1e6 / 1e12  # FP32 lanes x clock (non-FMA ops)
    fp32_peak_max = 148 * 128 * max_mhz * 1e6 / 1e12
    fp32_achieved = value * 1e6 * FLOPS_PER_CELL_UPDATE / world / 1e12
    devices_used = len(set(ring_devices)) if ring is not None else world
    if ring is not None:
        fp32_achieved = value * 1e6 * FLOPS_PER_CELL_UPDATE / devices_used / 1e12
    # Measured DRAM traffic of the dominant kernel (committed ncu capture of
    # one launch of this size) over the live average launch time.
    dram = None
    if traffic:
        dram_gbs = traffic / avg_launch_s / 1e9
        dram = {"achieved_gbs": round(dram_gbs, 1), "frac": round(dram_gbs / peaks["hbm_gbs"], 4),
                "bytes_per_cell_update": round(traffic / (per_rank_cells * levels), 3),
                "basis": "ncu dram__bytes_read.sum + dram__bytes_write.sum of one launch "
                         "(profiles/ncu_summary.json) / live average launch time"}
    # The binding roof leads: with K-level temporal blocking the stencil is
    # FP32-pipe bound (CUDA cores; the path is not a contraction, so no tensor
    # cores), so `achieved` is algorithmic FP32 ops per launch / launch time
    # and `peak` the FP32 lane peak at the board's maximum SM clock.  The HBM
    # view (compulsory bytes of a K-level block, the 16 B/cell-update
    # effective figure, and ncu-measured DRAM bytes) is nested under `hbm`.
    compulsory_bytes = BYTES_PER_CELL_UPDATE * per_rank_cells  # read + write u, v once per K-level block
    hbm = {"compulsory_gbs": round(compulsory_bytes / avg_launch_s / 1e9, 1),
           "compulsory_frac": round(compulsory_bytes / avg_launch_s / 1e9 / peaks["hbm_gbs"], 4),
           "effective_gbs": round(achieved_gbs, 1),
           "peak_gbs": peaks["hbm_gbs"],
           "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured" else "fallback",
           "basis": (f"compulsory = 16 B x cells per {levels}-level block (read u,v + write u,v once) / avg block "
                     f"time; effective = 16 B x cell-updates / time (what an unblocked kernel would have to "
                     f"move; > peak by design)"),
           **({"dram": dram} if dram else {})}
    roofline = {
        "bound": "fp32", "achieved": round(fp32_achieved, 2), "peak": round(fp32_peak_max, 2),
        "unit": "TFLOP/s", "frac": round(fp32_achieved / fp32_peak_max, 4), "traffic": traffic,
        "peak_source": (f"derived: 148 SM x 128 FP32 lanes x sm_max {max_mhz:.0f} MHz (MEASURED_PEAKS.json "
                        "sm_max_mhz; the file has no FP32 entry); tools/ubench_f32x2.cu measured 35.7-36.9 T "
                        "lane-ops/s of FFMA/FADD on this part"),
        "frac_at_median_clock": round(fp32_achieved / fp32_peak_tops, 4),
        "median_clock_mhz": round(sm_mhz),
        "note": (f"27 FP32 ops per cell-update (reference arithmetic); strict issues 25 on periodic lattices "
                 f"(fused -4*u_c and -4*v_c tails, gated 2-op x/3, Dv*lap_v skipped when Dv == 1; DESIGN.md "
                 f"section 4) "
                 f"x cell-updates per {levels}-level launch / avg launch time ({avg_launch_s * 1e6:.1f} us over "
                 f"{blocks_per_rank} blocks, {launches} launches); traffic = ncu DRAM bytes of one launch; "
                 "instruction-level account in profiles/sass_r02_wavefront_k4_classes.txt"),
        "hbm": hbm,
    }

    # ---- end to end through the public API with host buffers (N=1 only) ----
    e2e = None
    e2e_steps = args.e2e_steps or wl.e2e_steps
    if wl.name == "cfg4":
        # The whole sweep through the public API: the cells' initial states
        # uploaded from pinned host memory, S iterations with nssp=5 device
        # snapshots, the regime classifier on the device, the cells' final u
        # planes and labels back to the host (paper_2102_10340_b200.sweep.sweep_grid).
        from paper_2102_10340_b200.sweep import SweepSpec, sweep_grid
        cells = wl.rows_global * n
        u_in = torch.empty(wl.batch, cells, dtype=torch.float32).pin_memory()
        v_in = torch.empty(wl.batch, cells, dtype=torch.float32).pin_memory()
        st = fhn.init_center_square(wl.rows_global, n, 42)
        u_in[:] = torch.from_numpy(st.u)
        v_in[:] = torch.from_numpy(st.v)
        xs, ys = wl.axes()
        g7 = wl.gene7
        spec = SweepSpec(x_param="du", x_values=xs, y_param="dv", y_values=ys,
                         base_gene=fhn.Gene(dt=g7[0], a=g7[1], b=g7[2], eps=g7[3], c=g7[4], Du=g7[5], Dv=g7[6]),
                         base_config=fhn.RunConfig(init_mode=1, nn=wl.rows_global, nm=n, iter_max=S,
                                                   nssp=5 if S % 5 == 0 else 1, seed=42))
        sim.close()  # the sweep makes its own batched handle
        # One untimed sweep: the batched handle it creates (device state and
        # snapshot frames) is kept for the next sweep of the same shape, as
        # every other e2e here runs on warmed handles.
        sweep_grid(spec, device=local_rank, levels=args.levels, initial=(u_in.numpy(), v_in.numpy()))
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            res = sweep_grid(spec, device=local_rank, levels=args.levels, initial=(u_in.numpy(), v_in.numpy()))
        torch.cuda.synchronize()
        te = torch.tensor([time.perf_counter() - t0], device=red_dev)
        if dist is not None:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_s = float(te.item())
        e2e = {"value": round(cells * wl.batch * world * S * e2e_steps / e2e_s / 1e6, 2),
               "unit": "Mcell-updates/s", "h2d_bytes_per_step": 2 * 4 * cells * wl.batch * world,
               "d2h_bytes_per_step": (4 * cells * wl.batch + 8 * wl.batch + len(res.labels_csv)) * world,
               "path": "paper_2102_10340_b200.sweep.sweep_grid(spec, initial=host states): upload, advance with "
                       "nssp device snapshots, device classifier statistics and digests, the cells' final u "
                       "planes (what the reference keeps per cell, sweep.hpp:318) + labels CSV back"
                       + ("; per rank, max wall time over ranks" if world > 1 else ""),
               "steps": e2e_steps, "lattices_in_flight": wl.batch}
        if any(c.blew_up for c in res.cells):
            raise RuntimeError("blow-up in the cfg4 sweep")
    elif ring is not None:
        # The whole torus through the public Ring API from pinned host
        # memory: upload (split into the slabs) -> advance -> download.
        cells = wl.rows_global * n
        u_h = torch.empty(cells, dtype=torch.float32).pin_memory()
        v_h = torch.empty(cells, dtype=torch.float32).pin_memory()
        ring.download_ptr(u_h.data_ptr(), v_h.data_ptr())
        dev_ms = 0.0
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            ring.upload_ptr(u_h.data_ptr(), v_h.data_ptr())
            bad = ring.advance(S)
            dev_ms += ring.elapsed_ms()
            ring.download_ptr(u_h.data_ptr(), v_h.data_ptr())
            if bad.any():
                raise RuntimeError(f"blow-up in e2e ring run at iteration {int(bad[0])}")
        e2e_s = time.perf_counter() - t0
        e2e = {"value": round(cells * S * e2e_steps / e2e_s / 1e6, 2),
               "unit": "Mcell-updates/s", "h2d_bytes_per_step": 2 * 4 * cells,
               "d2h_bytes_per_step": 2 * 4 * cells,
               "path": "paper_2102_10340_b200.Ring: rdcnn_ring_upload (pinned host, split into the slabs) -> "
                       "rdcnn_ring_advance -> rdcnn_ring_download",
               "steps": e2e_steps, "lattices_in_flight": 1,
               "wall_ms_per_step": round(e2e_s * 1e3 / e2e_steps, 3),
               "device_ms_per_step": round(dev_ms / e2e_steps, 3),
               "copy_and_host_ms_per_step": round((e2e_s * 1e3 - dev_ms) / e2e_steps, 3)}
    elif not use_slab and wl.typ == 3 and not args.e2e_states:
        # Edge detection over a stream of images (the CeNN image-processing
        # mode): per image its 8-bit pixels go up from pinned host memory, the
        # device builds u = v = ka*x (init.hpp:58), advances S iterations and
        # normalises the final u plane with its own min/max (frame.hpp:28-44)
        # into the 8-bit edge map that comes back -- the reference CLI's
        # image in, frames out.  Several images in flight on alternating
        # handles, as for the state stream below.
        cells = wl.rows_global * n
        depth = max(1, min(args.e2e_depth or wl.e2e_depth, e2e_steps))
        px = torch.from_numpy(np.ascontiguousarray(wl.pixels()).reshape(-1)).pin_memory()
        outs = [torch.empty(cells, dtype=torch.uint8).pin_memory() for _ in range(depth)]
        pipe = fhn.Pipeline(wl.rows_global, n, depth=depth, sims=[sim], device=local_rank, mode=args.mode,
                            levels=args.levels, seg_rows=args.seg_rows)
        pipe.set_params(gene)
        for k, extra in enumerate(pipe.sims):  # first-use costs (graph capture, staging) stay out of the region
            if k > 0:
                extra.init_image_ptr(px.data_ptr(), 1.0)
                extra.advance(S)
            extra.frame_normalize_auto_ptr(outs[0].data_ptr())
        jobs = [(px.data_ptr(), outs[i % depth].data_ptr()) for i in range(e2e_steps)]
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        bad = pipe.run_images(jobs, S, 1.0)
        torch.cuda.synchronize()
        te = torch.tensor([time.perf_counter() - t0], device=red_dev)
        if dist is not None:  # replicas: max wall time over ranks
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        dev_ms = float(np.sum(pipe.last_device_ms))
        pipe.close()
        e2e_s = float(te.item())
        e2e = {"value": round(cells * world * S * e2e_steps / e2e_s / 1e6, 2),
               "unit": "Mcell-updates/s", "h2d_bytes_per_step": cells * world,
               "d2h_bytes_per_step": (cells + 16) * world,
               "path": (f"paper_2102_10340_b200.Pipeline(depth={depth}).run_images: per image "
                        "rdcnn_sim_init_image (8-bit pixels, pinned host) -> rdcnn_sim_advance -> "
                        "rdcnn_sim_frame_normalize_auto (final u plane -> 8-bit edge map + its min/max)"
                        + (", images on alternating handles so copies overlap advances" if depth > 1 else "")
                        + ("; per rank, max wall time over ranks" if world > 1 else "")),
               "steps": e2e_steps, "lattices_in_flight": depth,
               "wall_ms_per_step": round(e2e_s * 1e3 / e2e_steps, 3),
               "device_ms_per_step": round(dev_ms / e2e_steps, 3)}
        if bad.any():
            raise RuntimeError("blow-up in the e2e image stream")
    elif not use_slab:
        # A stream of independent lattices through the public Pipeline API:
        # each one is uploaded from pinned host memory, advanced S iterations
        # and downloaded; with depth 2 one lattice's copies overlap another's
        # advance.  Input: the state the timed run produced.
        cells = wl.rows_global * n
        depth = max(1, min(args.e2e_depth or wl.e2e_depth, e2e_steps))
        pinned = (1 + depth) * 2 * 4 * cells
        try:
            import psutil
            if depth > 1 and pinned > psutil.virtual_memory().available // 4:
                depth = 1  # keep pinned host buffers under a quarter of free RAM
        except ImportError:
            pass
        u_in = torch.empty(cells, dtype=torch.float32).pin_memory()
        v_in = torch.empty(cells, dtype=torch.float32).pin_memory()
        outs = [(torch.empty(cells, dtype=torch.float32).pin_memory(),
                 torch.empty(cells, dtype=torch.float32).pin_memory()) for _ in range(depth)]
        sim.download_ptr(u_in.data_ptr(), v_in.data_ptr())
        pipe = fhn.Pipeline(wl.rows_global, n, depth=depth, sims=[sim], device=local_rank, mode=args.mode,
                            levels=args.levels, seg_rows=args.seg_rows)
        pipe.set_params(gene)
        for extra in pipe.sims[1:]:  # first-use costs (incl. the graph capture) stay out of the timed region
            extra.upload_ptr(u_in.data_ptr(), v_in.data_ptr())
            extra.advance(S)
        jobs = [(u_in.data_ptr(), v_in.data_ptr(), outs[i % depth][0].data_ptr(), outs[i % depth][1].data_ptr())
                for i in range(e2e_steps)]
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        bad = pipe.run(jobs, S)
        torch.cuda.synchronize()
        te = torch.tensor([time.perf_counter() - t0], device=red_dev)
        if dist is not None:  # replicas: max wall time over ranks
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        dev_ms = float(np.sum(pipe.last_device_ms))
        pipe.close()
        e2e_s = float(te.item())
        split = {"wall_ms_per_step": round(e2e_s * 1e3 / e2e_steps, 3),
                 "device_ms_per_step": round(dev_ms / e2e_steps, 3)}
        if depth == 1:  # strictly sequential: the rest is the copies (and host calls)
            split["copy_and_host_ms_per_step"] = round((e2e_s * 1e3 - dev_ms) / e2e_steps, 3)
        e2e = {"value": round(cells * world * S * e2e_steps / e2e_s / 1e6, 2),
               "unit": "Mcell-updates/s", "h2d_bytes_per_step": 2 * 4 * cells * world,
               "d2h_bytes_per_step": 2 * 4 * cells * world,
               "path": (f"paper_2102_10340_b200.Pipeline(depth={depth}): per lattice rdcnn_sim_upload "
                        "(pinned host) -> rdcnn_sim_advance -> rdcnn_sim_download"
                        + (", lattices on alternating handles so copies overlap advances" if depth > 1 else "")
                        + ("; per rank, max wall time over ranks" if world > 1 else "")),
               "steps": e2e_steps, "lattices_in_flight": depth, **split}
        if bad.any() or not all(np.isfinite(u.numpy()).all() for u, _ in outs):
            raise RuntimeError("non-finite state after e2e")
    else:
        # Slab path: every rank uploads its slab from pinned host memory,
        # refills the ring's ghosts, advances, downloads; max over ranks.
        lib = fhn.load()
        cells = slab.rows * n
        u_h = torch.empty(cells, dtype=torch.float32).pin_memory()
        v_h = torch.empty(cells, dtype=torch.float32).pin_memory()
        fhn._lib.check(lib.rdcnn_sim_download(slab._h, u_h.data_ptr(), v_h.data_ptr()))
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        dev_ms = 0.0
        for _ in range(e2e_steps):
            fhn._lib.check(lib.rdcnn_sim_upload(slab._h, u_h.data_ptr(), v_h.data_ptr()))
            slab.fill_ghosts()
            bad = slab.advance(S)
            dev_ms += slab.elapsed_ms()
            fhn._lib.check(lib.rdcnn_sim_download(slab._h, u_h.data_ptr(), v_h.data_ptr()))
            if bad:
                raise RuntimeError(f"blow-up in e2e slab run near iteration {bad}")
        torch.cuda.synchronize()
        te = torch.tensor([time.perf_counter() - t0], device=red_dev)
        if dist is not None:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_s = float(te.item())
        e2e = {"value": round(cells * world * S * e2e_steps / e2e_s / 1e6, 2),
               "unit": "Mcell-updates/s", "h2d_bytes_per_step": 2 * 4 * cells * world,
               "d2h_bytes_per_step": 2 * 4 * cells * world,
               "path": "per rank: rdcnn_sim_upload (pinned host) -> rdcnn_slab_fill_ghosts -> "
                       "rdcnn_slab_advance -> rdcnn_sim_download; max wall time over ranks",
               "steps": e2e_steps, "wall_ms_per_step": round(e2e_s * 1e3 / e2e_steps, 3),
               "device_ms_per_step (rank 0)": round(dev_ms / e2e_steps, 3)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_sample(wl, args.cpu_seconds)
        except Exception as e:  # noqa: BLE001 - report, never hide
            cpu = {"value": None, "unit": "Mcell-updates/s", "cores": None, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    published, vs_basis = wl.published()
    vs_baseline = round(value / published, 2) if published else None
    if rank == 0:
        line = {
            "metric": "Mcell-updates/s", "value": round(value, 2), "unit": "Mcell-updates/s",
            "n_gpus": devices_used, "steps": args.steps, "warmup": args.warmup,
            **({"slabs": world, "devices": ring_devices} if ring is not None else {}),
            "ms_per_step": round(t_ms / args.steps, 3), "higher_is_better": True,
            "scaling": wl.scaling, "vs_baseline": vs_baseline, "dtype": "f32", "data": "synthetic",
            **({"vs_baseline_basis": vs_basis} if vs_basis else {}),
            "config": config_dict(wl, args, world, use_slab, transport),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clock_info,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
    ring_devices = None
    if "RANK" not in os.environ and (args.gpus > 1 or args.devices or args.ring):
        # Single-process multi-GPU: one process drives every slab through the
        # in-process ring (rdcnn_ring_*), one host thread per device.
        ring_devices = ([int(d) for d in args.devices.split(",")] if args.devices
                        else list(range(args.gpus)))
        world = len(ring_devices)
    if args.impl == "reference":
        bench_reference(args, rank, world)
        return
    bench_ours(args, rank, world, local_rank, ring_devices)


if __name__ == "__main__":
    main()
