"""One-off validation beyond 2^31 cells: a 49152^2 torus (2.4e9 cells, 38 GB
double-buffered on the device) for a few iterations on the B200, against the
reference's own parallel backend (oracle/_ref) on the host cores."""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2102_10340_b200 as fhn  # noqa: E402
from oracle.oracle import DEFAULT_GENE7, Reference  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 49152
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 8
t0 = time.time()
with fhn.Simulator(n, n) as sim:
    sim.init(2, 42)
    assert int(sim.advance(iters)[0]) == 0
    ms = sim.elapsed_ms()
    u, v = sim.download()
gpu = fhn.checksum(fhn.GridState(n, n, u, v))
print(f"gpu {n}^2 x{iters}: {gpu:016x} ({n * n * iters / ms / 1e3:.0f} Mcell-updates/s device; {time.time() - t0:.0f} s)",
      flush=True)
del u, v
ref = Reference()
u, v = ref.init(2, n, n, 42)
u, v, bad, sec = ref.run_timed(n, n, u, v, iters, DEFAULT_GENE7, backend="parallel")
want = ref.checksum(n, n, u, v)
print(f"reference {want:016x} ({ref.max_threads()} threads, {sec:.0f} s); match: {want == gpu}")
sys.exit(0 if want == gpu else 1)
