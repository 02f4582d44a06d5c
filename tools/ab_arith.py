"""Interleaved A/B of the strict arithmetic instances on one lattice (device
Mcell-updates/s): RDCNN_DIV3=3 (3-op x/3), =2 (2-op x/3, Dv product kept),
unset (automatic: 2-op x/3 and, with Dv == 1, the Dv product skipped).
Each pin gets a fresh handle (the variable is read at handle creation) and
runs long enough to reach the board's sustained (power-capped) clock."""
import argparse
import os
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2102_10340_b200 as fhn  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=4096)
ap.add_argument("--cols", type=int, default=4096)
ap.add_argument("--iters", type=int, default=20000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--pins", default="2,auto")
ap.add_argument("--persistent", type=int, default=-1)
a = ap.parse_args()
res = {}
for rep in range(a.reps):
    for pin in a.pins.split(","):
        if pin == "auto":
            os.environ.pop("RDCNN_DIV3", None)
        else:
            os.environ["RDCNN_DIV3"] = pin
        with fhn.Simulator(a.rows, a.cols, levels=4, persistent=a.persistent) as sim:
            sim.set_params(fhn.Gene(a=-0.05))
            sim.init(1, 42)
            sim.advance(max(a.iters // 4, 4))
            sim.advance(a.iters)
            ms = sim.elapsed_ms()
            v = a.rows * a.cols * a.iters / ms / 1e3
            res.setdefault(pin, []).append(v)
            print(f"rep {rep} pin={pin}: {v:,.0f} Mcell-updates/s ({ms:.1f} ms, {sim.launch_count()} launches)",
                  flush=True)
for pin, vs in res.items():
    print(f"pin={pin}: best {max(vs):,.0f} median {sorted(vs)[len(vs) // 2]:,.0f}")
