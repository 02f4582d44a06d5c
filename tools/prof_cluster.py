"""One 256^2 cluster-kernel advance (cfg1 shape) for ncu."""
import os
import sys

sys.path.insert(0, os.getcwd())
import paper_2102_10340_b200 as fhn  # noqa: E402

with fhn.Simulator(256, 256, 1, levels=4, persistent=1) as sim:
    sim.init(1, 42)
    sim.advance(1000)
    sim.advance(1000)
