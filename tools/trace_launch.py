"""Per-warp timeline of one wavefront launch (globaltimer start/end + SM id):
ramp-up, per-SM spread and tail.  python tools/trace_launch.py [rows cols levels]"""
import ctypes
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2102_10340_b200 as fhn  # noqa: E402

rows, cols, levels = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 4096, 4)))
lib = fhn.load()
with fhn.Simulator(rows, cols, levels=levels, persistent=-1) as sim:
    sim.set_params(fhn.Gene(a=-0.05))
    sim.init(1, 42)
    sim.advance(400)
    cap = 1 << 20
    buf = (ctypes.c_ulonglong * (3 * cap))()
    n = ctypes.c_longlong()
    for _ in range(3):
        fhn._lib.check(lib.rdcnn_sim_trace_launch(sim._h, levels, buf, cap, ctypes.byref(n)))
t = np.frombuffer(buf, dtype=np.uint64, count=3 * n.value).reshape(-1, 3).astype(np.float64)
import os  # noqa: E402
os.makedirs("gpurun_out", exist_ok=True)
np.save(f"gpurun_out/trace_{rows}x{cols}_k{levels}.npy", t)
t0 = t[:, 0].min()
st, en, sm = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, t[:, 2].astype(int)
dur = en - st
T = en.max()
print(f"{rows}x{cols} K={levels}: {n.value} warps on {len(set(sm))} SMs, launch span {T:.1f} us")
print(f"start: median {np.median(st):.2f} us, p99 {np.percentile(st, 99):.2f}, max {st.max():.2f}")
print(f"warp duration: min {dur.min():.1f} median {np.median(dur):.1f} p90 {np.percentile(dur, 90):.1f} max {dur.max():.1f} us")
# warp-slot occupancy over time: busy warp-us / (slots x span)
slots = 16 * len(set(sm))
print(f"busy warp-time / (slots x span) = {dur.sum() / (slots * T):.3f}")
per_sm_end = np.array([en[sm == k].max() for k in sorted(set(sm))])
per_sm_busy = np.array([dur[sm == k].sum() / (16 * en[sm == k].max()) for k in sorted(set(sm))])
print(f"SM last-warp end: min {per_sm_end.min():.1f} median {np.median(per_sm_end):.1f} max {per_sm_end.max():.1f} us")
print(f"per-SM slot utilisation to its own end: min {per_sm_busy.min():.3f} median {np.median(per_sm_busy):.3f}")
# same-SM spread of full-length warps
full = dur > 0.5 * np.median(dur)
spread = [dur[(sm == k) & full].max() / dur[(sm == k) & full].min() for k in sorted(set(sm)) if ((sm == k) & full).sum() > 1]
print(f"same-SM duration spread (max/min, full-length warps): median {np.median(spread):.3f} max {max(spread):.3f}")
hist, edges = np.histogram(en, bins=10, range=(0, T))
print("warp end-time histogram (10 bins over the span):", hist.tolist())
