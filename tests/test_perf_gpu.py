"""Throughput floors on the B200 (the reference's acceptance criterion 9 in
spirit: acceptance_main.cpp:279-288 asserts >= 200 Mcells/s for its CPU
backend).  Each floor is ~60 % of the measured rate (profiles/README.md), low
enough that the board's power cap never trips it, high enough that a kernel
or launch-path regression that keeps the results bit-exact still fails."""
import pytest

import paper_2102_10340_b200 as fhn

pytestmark = pytest.mark.gpu

# (rows, cols, batch, iterations per advance, floor in Mcell-updates/s, path)
CASES = [
    (4096, 4096, 1, 2000, 500_000, "wavefront, chip-filling (measured 780-835k)"),
    (1024, 1024, 1, 8000, 240_000, "wavefront, latency-bound with graph replay (measured 400k)"),
    (256, 256, 1, 1000, 48_000, "one-launch cluster kernel (measured 80-84k)"),
    (128, 128, 4096, 500, 550_000, "batched 128^2 sweep lattices (measured 930k)"),
]


@pytest.mark.parametrize("rows,cols,batch,iters,floor,path", CASES, ids=[c[5].split(",")[0] + f"-{c[0]}" for c in CASES])
def test_throughput_floor(rows, cols, batch, iters, floor, path):
    with fhn.Simulator(rows, cols, batch=batch) as sim:
        sim.set_params(fhn.Gene(a=-0.05))
        sim.init(1, 42)
        sim.advance(iters)  # warm-up: tuning, graph capture
        best = min((sim.advance(iters), sim.elapsed_ms())[1] for _ in range(3))
    rate = rows * cols * batch * iters / best / 1e3
    print(f"{rows}x{cols} x{batch}: {rate:,.0f} Mcell-updates/s ({path})")
    assert rate >= floor, f"{rate:,.0f} < floor {floor:,} Mcell-updates/s ({path})"
