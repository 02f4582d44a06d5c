"""Sweep fusion depth / segment height for one lattice and print device Mcells/s."""
import argparse
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2102_10340_b200 as fhn  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=4096)
ap.add_argument("--cols", type=int, default=4096)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--iters", type=int, default=2000)
ap.add_argument("--levels", default="1,2,4,8")
ap.add_argument("--segs", default="0")
ap.add_argument("--mode", default="strict")
ap.add_argument("--precision", default="single", choices=("single", "double"))
ap.add_argument("--lib", default=None, help="load this build of the extension instead (A/B runs)")
a = ap.parse_args()
if a.lib:
    fhn._lib.load(a.lib)
for lv in [int(x) for x in a.levels.split(",")]:
    for sg in [int(x) for x in a.segs.split(",")]:
        if a.precision == "double" and lv > 4:
            continue
        with fhn.Simulator(a.rows, a.cols, a.batch, levels=lv, seg_rows=sg, mode=a.mode,
                           precision=a.precision, persistent=-1) as sim:
            sim.set_params(fhn.Gene(a=-0.05))
            sim.init(1, 42)
            sim.advance(max(a.iters // 4, lv))
            sim.advance(a.iters)
            ms = sim.elapsed_ms()
            cu = a.rows * a.cols * a.batch * a.iters
            print(f"rows={a.rows} cols={a.cols} batch={a.batch} levels={lv} seg={sg} mode={a.mode} {a.precision}: "
                  f"{cu / ms / 1e3:,.0f} Mcells/s  ({ms:.1f} ms, {sim.launch_count()} launches)", flush=True)
