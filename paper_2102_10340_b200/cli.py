"""Command-line front end on the cuda backend (reference
proj/tools/rdcnn_cli.cpp): ``simulate``, ``bench`` and ``sweep`` with the
reference's flags, stdout lines, output files and exit codes
(0 ok, 1 invalid flags/config, 2 blow-up, 3 I/O).

  python -m paper_2102_10340_b200 simulate --typ 1 --size 64 --iters 200 --nssp 5 --seed 42

Differences, by scope: the montage/panel PNGs need the reference's bitmap
font renderer (out of scope); ``simulate`` writes one PGM per
snapshot instead, and ``sweep`` writes labels.csv and the per-cell PGMs.
Frames are min-max normalised to 8 bits on the device before download.
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import sys
import time
from typing import List, Optional, Tuple


from . import engine
from .engine import BlowUpError, Gene, GridState, RunConfig, Simulator, checksum, checksum_hex, validate_config
from .imageio import load_image_u8, write_pgm, write_png
from .sweep import ClassifierConfig, SweepSpec, format_double, sweep_grid

EXIT_OK, EXIT_INVALID, EXIT_BLOWUP, EXIT_IO = 0, 1, 2, 3

GENE_FLAGS = [("a", "a"), ("b", "b"), ("eps", "eps"), ("c", "c"), ("du", "Du"), ("dv", "Dv"), ("dt", "dt"),
              ("ka", "ka")]


def default_out_dir() -> str:
    return "out/" + datetime.datetime.now().strftime("%Y%m%d-%H%M%S")


# ---- manifest (config.hpp:97-190) ---------------------------------------------

def manifest_text(g: Gene, cfg: RunConfig, backend: str = "cuda") -> str:
    lines = [f"{k} = {format_double(getattr(g, attr))}" for k, attr in GENE_FLAGS]
    lines += [f"typ = {cfg.init_mode}", f"nn = {cfg.nn}", f"nm = {cfg.nm}", f"iter_max = {cfg.iter_max}",
              f"nssp = {cfg.nssp}", f"seed = {cfg.seed}", f"backend = {backend}", f"precision = {cfg.precision}"]
    if cfg.init_mode == 3 and cfg.image_path:
        lines.append(f"image = {cfg.image_path}")
    if cfg.init_mode == 3 and cfg.image_size:
        lines.append(f"image_size = {cfg.image_size}")
    return "\n".join(lines) + "\n"


def parse_manifest(text: str) -> Tuple[Gene, RunConfig]:
    kv = {}
    for line in text.splitlines():
        if not line or line.startswith("#"):
            continue
        if "=" not in line:
            raise ValueError(f"manifest line without '=': {line}")
        k, v = line.split("=", 1)
        kv[k.strip(" \t")] = v.strip(" \t\r")

    def need(k):
        if k not in kv:
            raise ValueError(f"manifest missing key: {k}")
        return kv[k]

    g = Gene(**{attr: float(need(k)) for k, attr in GENE_FLAGS})
    cfg = RunConfig(init_mode=int(need("typ")), nn=int(need("nn")), nm=int(need("nm")),
                    iter_max=int(need("iter_max")), nssp=int(need("nssp")), seed=int(need("seed")),
                    precision=need("precision"))
    if cfg.init_mode not in (1, 2, 3):
        raise ValueError("typ must be 1, 2 or 3")
    if need("backend") not in ("cuda", "reference", "shift", "blocked", "parallel"):
        raise ValueError(f"unknown backend: {kv['backend']}")
    if "image" in kv:
        cfg.image_path = kv["image"]
    if "image_size" in kv:
        cfg.image_size = int(kv["image_size"])
    return g, cfg


# ---- flags -----------------------------------------------------------------------

def add_gene_flags(p: argparse.ArgumentParser):
    d = Gene()
    for k, attr in GENE_FLAGS:
        p.add_argument(f"--{k}", type=float, default=getattr(d, attr))


def add_sim_flags(p: argparse.ArgumentParser):
    p.add_argument("--typ", type=int, default=1, choices=(1, 2, 3))
    p.add_argument("--size", type=int, default=512)
    p.add_argument("--rows", type=int, default=0)
    p.add_argument("--cols", type=int, default=0)
    p.add_argument("--image", default="")
    p.add_argument("--image-size", type=int, default=0)
    p.add_argument("--iters", type=int, default=10000)
    p.add_argument("--nssp", type=int, default=5)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--backend", default="cuda")
    p.add_argument("--precision", default="single", choices=("single", "double"))
    p.add_argument("--mode", default="strict", choices=("strict", "fast"))
    p.add_argument("--levels", type=int, default=4, choices=(1, 2, 4, 8))
    p.add_argument("--device", type=int, default=0)
    p.add_argument("--threads", type=int, default=0)
    p.add_argument("--tile-rows", type=int, default=64)
    p.add_argument("--tile-cols", type=int, default=64)
    p.add_argument("--out", default="")
    add_gene_flags(p)


def to_config(a) -> Tuple[Gene, RunConfig]:
    g = Gene(**{attr: getattr(a, k) for k, attr in GENE_FLAGS})
    engine.make_backend(a.backend, a.tile_rows, a.tile_cols, a.threads)  # raises on CPU kinds
    cfg = RunConfig(init_mode=a.typ, nn=a.rows if a.rows > 0 else a.size, nm=a.cols if a.cols > 0 else a.size,
                    image_path=a.image or None, image_size=a.image_size or None, iter_max=a.iters,
                    nssp=a.nssp, seed=a.seed, precision=a.precision)
    return g, cfg


def report_validation(issues: List[str]) -> int:
    for issue in issues:
        kind, msg = issue.split(": ", 1)
        print(f"error [{kind}]: {msg}", file=sys.stderr)
    return EXIT_INVALID


def advisory(g: Gene):
    if g.dt * max(g.Du, g.Dv) > 0.25:
        print(f"advisory: dt*max(Du,Dv) = {format_double(g.dt * max(g.Du, g.Dv))} exceeds 0.25; "
              "explicit Euler may be unstable", file=sys.stderr)


# ---- simulate ------------------------------------------------------------------

def simulate(g: Gene, cfg: RunConfig, out_dir: str, mode: str, levels: int, device: int) -> int:
    image = None
    try:
        if cfg.init_mode == 3:
            image = load_image_u8(cfg.image_path, cfg.image_size)
            cfg.nn, cfg.nm = image.shape
    except (OSError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_IO
    try:
        os.makedirs(out_dir, exist_ok=True)
        with open(os.path.join(out_dir, "manifest.txt"), "w") as f:
            f.write(manifest_text(g, cfg))
    except OSError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_IO

    print(f"FHN Calculation: {cfg.nn} x {cfg.nm} mesh", flush=True)
    sim = Simulator(cfg.nn, cfg.nm, device=device, mode=mode, levels=levels, precision=cfg.precision)
    sim.set_params(g)
    if cfg.init_mode == 3:
        sim.init_image(image, g.ka)
    else:
        sim.init(cfg.init_mode, cfg.seed)
    test_mod = cfg.iter_max // cfg.nssp
    sim.frames_reserve(cfg.nssp + 1)
    sim.frame_capture(0)
    t0 = time.perf_counter()
    done = 0
    for f in range(1, cfg.nssp + 1):
        bad = sim.advance(test_mod)
        if bad[0]:
            print(f"error: blow-up: non-finite state after iteration {done + int(bad[0])}", file=sys.stderr)
            return EXIT_BLOWUP
        done += test_mod
        sim.frame_capture(f)
        print(f"{done - 1}, (elapsed: {time.perf_counter() - t0:f} s)", flush=True)
    wall = time.perf_counter() - t0
    u, v = sim.download()
    cells = cfg.nn * cfg.nm * cfg.iter_max
    mn, mx, _ = sim.frame_stats(cfg.nssp)
    print(f"total: {wall:f} s")
    print("=====")
    print(f"per cell time: {format_double(wall * 1e9 / cells)} nano-seconds")
    print(f"speed: {format_double(cells / (wall * 1e6))} Mega cells/second")
    print(f"max-min= {mx[0] - mn[0]:f}")
    print(f"checksum= {checksum_hex(checksum(GridState(cfg.nn, cfg.nm, u, v)))}")
    print("=====", flush=True)
    try:
        for f in range(cfg.nssp + 1):
            fmn, fmx, _ = sim.frame_stats(f)
            write_pgm(os.path.join(out_dir, f"frame_{f * test_mod:06d}_u.pgm"),
                      sim.frame_normalize(f, 0, fmn[0], fmx[0]))
        fu = sim.frame_normalize(-1, 0, float(mn[0]), float(mx[0]))
        from .imageio import normalize_frame
        fv, _, _ = normalize_frame(v.reshape(cfg.nn, cfg.nm))  # v is not in the frame store
        for name, img in (("final_u", fu), ("final_v", fv)):
            write_pgm(os.path.join(out_dir, name + ".pgm"), img)
            write_png(os.path.join(out_dir, name + ".png"), img)
    except OSError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_IO
    sim.close()
    return EXIT_OK


def cmd_simulate(a) -> int:
    try:
        if a.manifest:
            with open(a.manifest) as f:
                g, cfg = parse_manifest(f.read())
        else:
            g, cfg = to_config(a)
    except (ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INVALID
    issues = validate_config(cfg, g)
    if issues:
        return report_validation(issues)
    advisory(g)
    return simulate(g, cfg, a.out or default_out_dir(), a.mode, a.levels, a.device)


# ---- bench (bench.hpp:96-253) ----------------------------------------------

def cmd_bench(a) -> int:
    g = Gene(**{attr: getattr(a, k) for k, attr in GENE_FLAGS})
    advisory(g)
    try:
        sizes = [int(s) for s in a.sizes.split(",") if s]
        for name in [b for b in a.backends.split(",") if b]:
            engine.make_backend(name)
        if not sizes:
            raise ValueError("need at least one backend and one size")
        if a.iters < 1 or a.reps < 1 or any(n < 11 for n in sizes):
            raise ValueError("bench needs iter_max >= 1, reps >= 1 and sizes >= 11")
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INVALID
    records = []
    warmed = False
    for n in sizes:
        with Simulator(n, n, mode=a.mode, levels=a.levels, precision=a.precision) as sim:
            sim.set_params(g)
            if not warmed:
                sim.init(1, a.seed)
                sim.advance(min(a.iters, 100))
                warmed = True
            times, digest = [], 0
            for _ in range(a.reps):
                sim.init(1, a.seed)
                t0 = time.perf_counter()
                bad = sim.advance(a.iters)
                times.append(time.perf_counter() - t0)
                if bad[0]:
                    print(f"error: blow-up in benchmark cell backend=cuda N={n} at iteration {int(bad[0])}",
                          file=sys.stderr)
                    return EXIT_BLOWUP
                u, v = sim.download()
                digest = checksum(GridState(n, n, u, v))
            sec = sorted(times)[len(times) // 2]
            work = float(n) * n * a.iters
            records.append(dict(backend="cuda", hardware=a.hardware, n=n, iters=a.iters, seconds=sec,
                                mcells_per_s=work / (sec * 1e6), ns_per_cell_iter=sec * 1e9 / work,
                                checksum=f"{digest:016x}"))
    print("backend  " + "  ".join(f"N={r['n']}" for r in records))
    print("cuda     " + "  ".join("%.5g (%.4g)" % (r["mcells_per_s"], r["seconds"]) for r in records))
    out_dir = a.out or default_out_dir()
    try:
        os.makedirs(out_dir, exist_ok=True)
        cfg = RunConfig(init_mode=1, nn=sizes[0], nm=sizes[0], iter_max=a.iters, nssp=1, seed=a.seed,
                        precision=a.precision)
        with open(os.path.join(out_dir, "manifest.txt"), "w") as f:
            f.write(manifest_text(g, cfg))
        with open(os.path.join(out_dir, "bench.csv"), "w") as f:
            f.write("backend,hardware,n,iters,seconds,mcells_per_s,ns_per_cell_iter,checksum\n")
            for r in records:
                f.write("%s,%s,%d,%d,%.5g,%.5g,%.5g,%s\n" % (r["backend"], r["hardware"], r["n"], r["iters"],
                                                           r["seconds"], r["mcells_per_s"],
                                                           r["ns_per_cell_iter"], r["checksum"]))
        if a.json:
            with open(os.path.join(out_dir, "bench.json"), "w") as f:
                json.dump(records, f, indent=2)
                f.write("\n")
    except OSError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_IO
    return EXIT_OK


# ---- sweep (sweep.hpp:255-350) ------------------------------------------------

def parse_axis(text: str):
    if ":" not in text:
        raise ValueError(f"axis spec must look like du:0.3,0.5 (got '{text}')")
    param, vals = text.split(":", 1)
    return param, [float(t) for t in vals.split(",") if t]


def cmd_sweep(a) -> int:
    try:
        if not a.x and not a.y:
            a.x, a.y = "a:-0.5,-0.4,-0.3,-0.2,-0.1,0,0.1", "b:0.9,1.1,1.3,1.5,1.7"
        if not a.x or not a.y:
            raise ValueError("--x and --y must be given together")
        xp, xs = parse_axis(a.x)
        yp, ys = parse_axis(a.y)
        g, cfg = to_config(a)
        cc = ClassifierConfig(a.homogeneity_rel, a.homogeneity_floor, a.activity_rel, a.growth_factor,
                              a.dip_tolerance)
        fixed = None
        if a.range:
            lo, hi = a.range.split(":")
            fixed = (float(lo), float(hi))
        spec = SweepSpec(xp, xs, yp, ys, base_gene=g, base_config=cfg, per_cell_seed=a.per_cell_seed,
                         parallel_cells=a.parallel_cells, fixed_range=fixed, classifier=cc)
        issues = validate_config(cfg, g)
        if cfg.init_mode == 3 and a.image:
            issues = [i for i in issues if not i.startswith("MissingImage")]
        if issues:
            return report_validation(issues)
        image = load_image_u8(cfg.image_path, cfg.image_size) if cfg.init_mode == 3 else None
    except (ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INVALID
    out_dir = a.out or default_out_dir()
    try:
        os.makedirs(out_dir, exist_ok=True)
        with open(os.path.join(out_dir, "manifest.txt"), "w") as f:
            f.write(manifest_text(g, cfg))
        devices = [int(d) for d in a.devices.split(",")] if a.devices else None
        res = sweep_grid(spec, image=image, device=a.device, levels=a.levels, devices=devices)
        with open(os.path.join(out_dir, "labels.csv"), "w") as f:
            f.write(res.labels_csv)
        from .imageio import normalize_frame
        for c in res.cells:
            if c.blew_up:
                continue
            img, _, _ = normalize_frame(c.final_u.reshape(res.rows, res.cols))
            write_pgm(os.path.join(out_dir, f"cell_{format_double(c.x_value)}_{format_double(c.y_value)}.pgm"), img)
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INVALID
    except OSError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_IO
    for yi in range(len(res.y_values)):
        for xi in range(len(res.x_values)):
            c = res.at(yi, xi)
            print(f"{xp}={format_double(c.x_value)} {yp}={format_double(c.y_value)} -> {c.outcome.label}")
    print(f"wrote {out_dir}/labels.csv and {len(res.cells)} cell frames")
    return EXIT_OK


def main(argv: Optional[List[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="rdcnn", description="Two-layer FitzHugh-Nagumo RD-CNN simulator (cuda)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("simulate", help="run one simulation")
    add_sim_flags(s)
    s.add_argument("--manifest", default="")
    s.add_argument("--band-timing", action="store_true")
    b = sub.add_parser("bench", help="benchmark sizes on the cuda backend")
    b.add_argument("--backends", default="cuda")
    b.add_argument("--sizes", default="128,256,512,1024,2048,4096")
    b.add_argument("--iters", type=int, default=10000)
    b.add_argument("--reps", type=int, default=3)
    b.add_argument("--seed", type=int, default=42)
    b.add_argument("--precision", default="single", choices=("single", "double"))
    b.add_argument("--hardware", default="b200")
    b.add_argument("--mode", default="strict", choices=("strict", "fast"))
    b.add_argument("--levels", type=int, default=4, choices=(1, 2, 4, 8))
    b.add_argument("--out", default="")
    b.add_argument("--json", action="store_true")
    add_gene_flags(b)
    w = sub.add_parser("sweep", help="explore a two-parameter plane")
    w.add_argument("--x", default="")
    w.add_argument("--y", default="")
    add_sim_flags(w)
    w.add_argument("--range", default="")
    w.add_argument("--per-cell-seed", action="store_true")
    w.add_argument("--devices", default="", help="comma-separated GPUs to split the cells over")
    w.add_argument("--parallel-cells", action="store_true")
    cc = ClassifierConfig()
    w.add_argument("--homogeneity-rel", type=float, default=cc.homogeneity_rel)
    w.add_argument("--homogeneity-floor", type=float, default=cc.homogeneity_floor)
    w.add_argument("--activity-rel", type=float, default=cc.activity_rel)
    w.add_argument("--growth-factor", type=float, default=cc.growth_factor)
    w.add_argument("--dip-tolerance", type=float, default=cc.dip_tolerance)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code == 0 else EXIT_INVALID
    try:
        if a.cmd == "simulate":
            return cmd_simulate(a)
        if a.cmd == "bench":
            return cmd_bench(a)
        return cmd_sweep(a)
    except BlowUpError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_BLOWUP


if __name__ == "__main__":
    sys.exit(main())
