"""Time small single lattices through both paths: the persistent cluster
kernel (one launch per advance) and the K-level wavefront kernel.
Usage: python tools/small_grid.py [rows cols iters ...]"""
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
import paper_2102_10340_b200 as fhn  # noqa: E402

cases = [(256, 256, 1000), (128, 128, 1000), (256, 128, 1000), (100, 256, 1000), (256, 256, 10000)]
if len(sys.argv) > 3:
    a = [int(x) for x in sys.argv[1:]]
    cases = [tuple(a[i:i + 3]) for i in range(0, len(a), 3)]
for rows, cols, iters in cases:
    out = []
    for pers, levels in ((1, 4), (-1, 1), (-1, 2), (-1, 4), (-1, 8)):
        try:
            with fhn.Simulator(rows, cols, levels=levels, persistent=pers) as sim:
                sim.init(1, 42)
                sim.advance(iters)  # warm-up
                best = min((sim.advance(iters), sim.elapsed_ms())[1] for _ in range(5))
        except fhn.RdcnnError as e:
            out.append(f"{'cluster' if pers == 1 else f'K={levels}'}: n/a ({e})")
            continue
        name = "cluster" if pers == 1 else f"K={levels}"
        out.append(f"{name}: {rows * cols * iters / best / 1e3:9.0f} Mcell-updates/s ({best:.3f} ms)")
    print(f"{rows}x{cols} x{iters}: " + " | ".join(out), flush=True)
