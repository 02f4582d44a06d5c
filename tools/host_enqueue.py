"""Host enqueue rate vs device time per launch of an advance (is the
per-launch path host-bound?  If so CUDA graphs would pay)."""
import sys, time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2102_10340_b200 as fhn
for n, it in ((512, 20000), (1024, 10000), (4096, 4000)):
    with fhn.Simulator(n, n, levels=4, persistent=-1) as sim:
        sim.set_params(fhn.Gene(a=-0.05)); sim.init(1, 42)
        sim.advance(it)
        t0 = time.perf_counter(); sim.advance(it); wall = time.perf_counter() - t0
        gpu = sim.elapsed_ms() / 1e3
        L = sim.launch_count()
        print(f"{n}^2 x{it}: {L} launches, GPU {gpu*1e3:.1f} ms ({gpu/L*1e6:.2f} us/launch), host wall {wall*1e3:.1f} ms", flush=True)
