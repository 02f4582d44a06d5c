"""Small runs of every kernel path, for compute-sanitizer (memcheck /
racecheck / synccheck): wavefront K=1/2/4/8 at W=1/4 (odd and full-width
shapes), batch with per-grid genes, fp64, fast mode, blow-up replay, the
fused peer-ring slab (world 1), the cluster kernel (incl. its rows-per-warp
trials), CUDA-graph capture and replay, concurrent handles from host threads
(engine.Pipeline), device
checksums and frame analysis."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2102_10340_b200 as fhn  # noqa: E402
from paper_2102_10340_b200.slab import SlabStepper  # noqa: E402

for rows, cols in ((17, 23), (40, 128), (64, 96)):
    for lv in (1, 2, 4, 8):
        with fhn.Simulator(rows, cols, levels=lv, persistent=-1) as s:
            s.init(2, 3)
            s.advance(2 * lv + 1)
with fhn.Simulator(32, 128, batch=5, levels=4) as s:
    s.set_params([fhn.Gene(Du=0.06 + 0.01 * k) for k in range(4)] + [fhn.Gene(dt=100.0)])
    s.init(1, 42)
    s.advance(40)
    s.checksums()
    s.frames_reserve(2)
    s.frame_capture(0)
    s.frame_stats(0)
with fhn.Simulator(24, 40, levels=4, precision="double") as s:
    s.init(2, 5)
    s.advance(11)
with fhn.Simulator(48, 64, levels=4, mode="fast") as s:
    s.init(2, 5)
    s.advance(11)
sl = SlabStepper(32, 128, rank=0, world=1, ghost=4, device=0)
sl.init(2, 7)
sl.fill_ghosts()
sl.advance(13)
sl.close()
with fhn.Simulator(64, 128, persistent=1) as s:  # cluster path
    s.init(2, 9)
    s.advance(20)
with fhn.Simulator(64, 128, persistent=1) as s:  # cluster path blow-up + re-run
    s.set_params(fhn.Gene(dt=100.0))
    s.init(2, 9)
    s.advance(20)
with fhn.Simulator(96, 96, persistent=-1) as s:  # CUDA-graph capture, then replay (under-filled launches)
    s.init(2, 4)
    s.advance(64)
    s.advance(64)
with fhn.Simulator(64, 128, persistent=1) as s:  # cluster rows-per-warp trials (>= 4 x 128 steps)
    s.init(2, 9)
    s.advance(520)
import numpy as np  # noqa: E402

st = fhn.init_full_random(40, 128, 5)
outs = [(np.empty(40 * 128, np.float32), np.empty(40 * 128, np.float32)) for _ in range(3)]
with fhn.Pipeline(40, 128, depth=2, persistent=-1) as p:  # two handles driven from two host threads
    p.run([(st.u.ctypes.data, st.v.ctypes.data, u.ctypes.data, v.ctypes.data) for u, v in outs], 9)
print("sanitize paths done")
