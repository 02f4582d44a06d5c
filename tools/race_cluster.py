"""The cluster kernel with several warps per CTA, one rows-per-warp variant
at a time (RDCNN_CLUSTER_RW), for compute-sanitizer racecheck."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2102_10340_b200 as fhn  # noqa: E402

rows, cols, steps = (int(x) for x in sys.argv[1:4])
with fhn.Simulator(rows, cols, persistent=1) as s:
    s.init(2, 9)
    s.advance(steps)
print("done", rows, cols, steps)
