"""Wall-time breakdown of the cfg4 parameter sweep (4096 x 128^2 x 5000
iterations, nssp 5) through sweep_grid, phase by phase (monkey-patched
timers around the Simulator calls)."""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2102_10340_b200 import sweep as sw  # noqa: E402
from paper_2102_10340_b200.engine import RunConfig, Simulator  # noqa: E402

T = {}


def timed(name, fn):
    def w(*a, **k):
        t0 = time.perf_counter()
        r = fn(*a, **k)
        T[name] = T.get(name, 0.0) + time.perf_counter() - t0
        return r
    return w


for name in ("advance", "frame_capture", "frame_stats", "frame_active", "download", "init", "set_params",
             "frames_reserve", "frame_download", "upload", "__init__", "close"):
    setattr(Simulator, name, timed(name, getattr(Simulator, name)))
sw.classify = timed("classify", sw.classify)
sw.labels_csv = timed("labels_csv", sw.labels_csv)
for name in ("checksums",):
    setattr(Simulator, name, timed(name, getattr(Simulator, name)))

side = int(sys.argv[1]) if len(sys.argv) > 1 else 64
# "initial": upload the cells' states from pinned host memory, as bench.py's cfg4 e2e does
initial = None
if len(sys.argv) > 2 and sys.argv[2] == "initial":
    import torch
    from paper_2102_10340_b200 import init_center_square
    st = init_center_square(128, 128, 42)
    u_in = torch.empty(side * side, 128 * 128, dtype=torch.float32).pin_memory()
    v_in = torch.empty(side * side, 128 * 128, dtype=torch.float32).pin_memory()
    u_in[:] = torch.from_numpy(st.u)
    v_in[:] = torch.from_numpy(st.v)
    initial = (u_in.numpy(), v_in.numpy())
cfg = RunConfig()
cfg.nn = cfg.nm = 128
cfg.iter_max = 5000
cfg.nssp = 5
spec = sw.SweepSpec("du", list(np.linspace(0.02, 0.70, side)), "dv", list(np.linspace(0.50, 1.20, side)),
                    base_config=cfg)
for rep in range(2):  # the second sweep is the one reported (first-use costs excluded)
    T.clear()
    t0 = time.perf_counter()
    res = sw.sweep_grid(spec, initial=initial)
    wall = time.perf_counter() - t0
labels = {}
for c in res.cells:
    labels[c.outcome.label] = labels.get(c.outcome.label, 0) + 1
print(f"sweep {side}x{side} cells of 128^2 x 5000: wall {wall:.3f} s; labels {labels}")
for k, v in sorted(T.items(), key=lambda x: -x[1]):
    print(f"  {k:15s} {v:.3f} s")
