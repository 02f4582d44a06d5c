import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2102_10340_b200 as fhn
sim = fhn.Simulator(256, 256, device=0, levels=4)
sim.set_params(fhn.Gene())
sim.init(1, 42)
for _ in range(3): sim.advance(1000)
stream = torch.cuda.ExternalStream(sim.stream(), device=0)
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda:0")
for use_flush in (False, True):
    ext, internal = [], []
    for _ in range(10):
        if use_flush:
            flush.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sim.advance(1000)
        e1.record(stream)
        torch.cuda.synchronize()
        ext.append(e0.elapsed_time(e1)); internal.append(sim.elapsed_ms())
    print(f"flush={use_flush}: external {sorted(ext)[5]:.4f} ms, internal {sorted(internal)[5]:.4f} ms, launches {sim.launch_count()}")
# host-side cost of advance
t = time.perf_counter()
for _ in range(20): sim.advance(1000)
print(f"wall per advance {(time.perf_counter() - t) / 20 * 1e3:.4f} ms")
