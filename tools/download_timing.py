import sys, os, time, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2102_10340_b200 as fhn
from paper_2102_10340_b200._lib import check
B = 4096
with fhn.Simulator(128, 128, batch=B, levels=4) as sim:
    sim.init(1, 42); sim.frames_reserve(2); sim.frame_capture(0)
    lib = sim._lib
    n = B * 128 * 128
    for rep in range(2):
        t = time.perf_counter(); u = np.empty(n, np.float32); check(lib.rdcnn_sim_frame_download(sim._h, 0, u.ctypes.data)); a = time.perf_counter() - t
        u2 = np.ones(n, np.float32)
        t = time.perf_counter(); check(lib.rdcnn_sim_frame_download(sim._h, 0, u2.ctypes.data)); b = time.perf_counter() - t
        p = torch.empty(n, dtype=torch.float32).pin_memory()
        t = time.perf_counter(); check(lib.rdcnn_sim_frame_download(sim._h, 0, p.data_ptr())); c = time.perf_counter() - t
        t = time.perf_counter(); u3 = np.empty(n, np.float32); u3[:] = p.numpy(); d = time.perf_counter() - t
        print(f"fresh {a*1e3:.1f} ms, touched {b*1e3:.1f} ms, pinned {c*1e3:.1f} ms, host copy pinned->fresh {d*1e3:.1f} ms")
