"""One small row-ring advance (RDCNN_ROWRING=2 must be set) for compute-sanitizer runs:
C=1 (M=8) and C=2 (M=4) rings, with a blow-up replay.

  RDCNN_ROWRING=2 RDCNN_RR_M=4 compute-sanitizer --tool racecheck python tools/sanitize_rowring.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_10340_b200 as fhn  # noqa: E402

with fhn.Simulator(40, 1024, 1, levels=4, mode="strict", persistent=-1) as sim:
    sim.set_params(fhn.Gene())
    sim.init(2, 42)
    sim.advance(12)
    print("checksum %016x" % int(sim.checksums()[0]))
with fhn.Simulator(40, 1024, 1, levels=4, mode="strict", persistent=-1) as sim:
    sim.set_params(fhn.Gene(dt=100.0))
    sim.init(2, 42)
    try:
        sim.advance(12)
    except Exception as e:  # the blow-up is the point
        print("blow-up:", e)
