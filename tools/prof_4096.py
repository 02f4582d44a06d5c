import sys, os
sys.path.insert(0, os.getcwd())
import paper_2102_10340_b200 as fhn
with fhn.Simulator(4096, 4096, 1, levels=4, mode="strict", persistent=-1) as sim:
    sim.set_params(fhn.Gene(a=-0.05))
    sim.init(1, 42)
    sim.advance(400)
