"""One short advance of a given lattice (for ncu captures).

  python tools/prof_shape.py ROWS COLS STEPS [LEVELS]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_10340_b200 as fhn  # noqa: E402

rows, cols, steps = (int(x) for x in sys.argv[1:4])
levels = int(sys.argv[4]) if len(sys.argv) > 4 else 4
with fhn.Simulator(rows, cols, 1, levels=levels, mode="strict", persistent=-1) as sim:
    sim.set_params(fhn.Gene(a=-0.05))
    sim.init(1, 42)
    sim.advance(steps)
    sim.advance(steps)
