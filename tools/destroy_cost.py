"""Time handle creation / destruction for a cfg4-sized batch (diagnostics)."""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2102_10340_b200 as fhn  # noqa: E402

for frames in (0, 6, 6, 6):
    t0 = time.perf_counter()
    sim = fhn.Simulator(128, 128, batch=4096)
    t1 = time.perf_counter()
    if frames:
        sim.frames_reserve(frames)
        sim.frame_capture(0)
    sim.init(1, 42)
    sim.advance(100)
    t2 = time.perf_counter()
    sim.close()
    t3 = time.perf_counter()
    print(f"frames={frames}: create {1e3 * (t1 - t0):.1f} ms, destroy {1e3 * (t3 - t2):.1f} ms", flush=True)

# The sweep's exact sequence (sweep._run_cells), then destroy.
import numpy as np  # noqa: E402

for rep in range(2):
    T = {}
    sim = fhn.Simulator(128, 128, batch=4096)
    t = time.perf_counter
    a = t(); sim.set_params([fhn.Gene(Du=0.02 + 0.0001 * k) for k in range(4096)]); T["set_params"] = t() - a
    a = t(); sim.init(1, 42); sim.frames_reserve(6); sim.frame_capture(0); T["init+reserve"] = t() - a
    a = t()
    for f in range(1, 6):
        sim.advance(1000)
        sim.frame_capture(f)
    T["advance"] = t() - a
    a = t(); st = [sim.frame_stats(f) for f in range(6)]; T["stats"] = t() - a
    a = t(); [sim.frame_active(f, st[f][2], np.full(4096, 0.1)) for f in range(6)]; T["active"] = t() - a
    a = t(); sim.checksums(); T["checksums"] = t() - a
    a = t(); fu = sim.frame_download(5); T["frame_download"] = t() - a
    a = t(); sim.close(); T["close"] = t() - a
    print("sweep sequence:", {k: round(v * 1e3, 1) for k, v in T.items()}, "ms", flush=True)
