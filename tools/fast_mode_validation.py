"""Statistical validation of the opt-in fast (FMA-contracted) mode against
strict, as SURVEY §7 prescribes ("activity curve / regime label, never
max-abs"): fast drifts from strict by O(1) after ~10^4 iterations on
slow-growth genes (FMA changes every rounding), so agreement is judged on
the outcomes the reference's analysis reports.

  python tools/fast_mode_validation.py [--cells 64] [--iters 5000] [--out profiles/fast_mode_r02.json]

1. cfg4 (BASELINE configs[3]): the Du x Dv sweep of 128^2 lattices, labels
   (sweep.hpp:73-112 classify_outcome) strict vs fast, cell by cell.
2. cfg2 (configs[1]): the 4096^2 slow-growth lattice, growth_curve
   (sweep.hpp:48-64) at every 1000 iterations to 10 000, strict vs fast,
   plus the final max |u_fast - u_strict| for the record.
"""
import argparse
import dataclasses
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2102_10340_b200 as fhn  # noqa: E402
from paper_2102_10340_b200.sweep import SweepSpec, sweep_grid  # noqa: E402


def sweep_labels(mode, n_side, iters):
    xs = list(np.linspace(0.02, 0.70, 64))
    ys = list(np.linspace(0.50, 1.20, 64))
    step = 64 // n_side
    xs, ys = xs[::step], ys[::step]
    be = fhn.make_backend("cuda", mode=mode)
    spec = SweepSpec(x_param="du", x_values=xs, y_param="dv", y_values=ys, base_gene=fhn.Gene(),
                     base_config=fhn.RunConfig(init_mode=1, nn=128, nm=128, iter_max=iters, nssp=5, seed=42,
                                               backend=be))
    t0 = time.perf_counter()
    res = sweep_grid(spec)
    return [c.outcome.label for c in res.cells], [c.outcome.activity_counts for c in res.cells], \
        time.perf_counter() - t0


def growth_curve(u, threshold):
    med = np.partition(u, u.size // 2)[u.size // 2]
    return int(np.count_nonzero(np.abs(u.astype(np.float64) - float(med)) > threshold))


def cfg2_curves(size, iters, every):
    g = fhn.Gene(a=-0.05)
    out = {}
    for mode in ("strict", "fast"):
        frames = []
        with fhn.Simulator(size, size, mode=mode) as sim:
            sim.set_params(g)
            sim.init(1, 42)
            frames.append(sim.download()[0])
            for _ in range(iters // every):
                assert int(sim.advance(every)[0]) == 0
                frames.append(sim.download()[0])
        out[mode] = frames
    # the reference's threshold: activity_rel x the final u range (of each run)
    curves = {}
    for mode, frames in out.items():
        rng = float(frames[-1].max() - frames[-1].min())
        curves[mode] = [growth_curve(f, 0.1 * rng) for f in frames]
    maxabs = float(np.max(np.abs(out["fast"][-1].astype(np.float64) - out["strict"][-1])))
    return curves, maxabs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=64, help="sweep side (64 = the full cfg4 plane)")
    ap.add_argument("--iters", type=int, default=5000)
    ap.add_argument("--cfg2-size", type=int, default=4096)
    ap.add_argument("--cfg2-iters", type=int, default=10000)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "fast_mode_r02.json"))
    a = ap.parse_args()
    ls, cs, ts = sweep_labels("strict", a.cells, a.iters)
    lf, cf, tf = sweep_labels("fast", a.cells, a.iters)
    diff = [i for i, (x, y) in enumerate(zip(ls, lf)) if x != y]
    rel = [abs(p - q) / max(1, p) for s_, f_ in zip(cs, cf) for p, q in zip(s_, f_)]
    curves, maxabs = cfg2_curves(a.cfg2_size, a.cfg2_iters, 1000)
    cs2, cf2 = curves["strict"], curves["fast"]
    rel2 = [abs(p - q) / max(1, p) for p, q in zip(cs2, cf2)]
    rep = {
        "cfg4_sweep": {"cells": len(ls), "iters": a.iters, "labels_differing": len(diff),
                       "agreement": 1 - len(diff) / len(ls),
                       "differing_cells": [{"index": i, "strict": ls[i], "fast": lf[i]} for i in diff[:20]],
                       "label_counts_strict": {k: ls.count(k) for k in sorted(set(ls))},
                       "label_counts_fast": {k: lf.count(k) for k in sorted(set(lf))},
                       "activity_count_rel_diff_max": max(rel) if rel else 0.0,
                       "activity_count_rel_diff_median": float(np.median(rel)) if rel else 0.0,
                       "seconds_strict": round(ts, 2), "seconds_fast": round(tf, 2)},
        "cfg2_growth_curve": {"size": a.cfg2_size, "every": 1000, "iters": a.cfg2_iters,
                              "strict": cs2, "fast": cf2, "rel_diff_per_frame": [round(x, 5) for x in rel2],
                              "rel_diff_max": max(rel2), "final_max_abs_u_diff": maxabs},
    }
    with open(a.out, "w") as f:
        json.dump(rep, f, indent=1)
    print(json.dumps({k: {kk: vv for kk, vv in v.items() if kk != "differing_cells"} for k, v in rep.items()},
                     indent=1))


if __name__ == "__main__":
    main()
