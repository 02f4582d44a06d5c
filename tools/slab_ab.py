"""A/B of the cfg5 lattice on one GPU: periodic handle vs world-1 slab ring
with and without the exact-blow-up checkpoint tee (device ms per 100-step
advance, alternating passes)."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2102_10340_b200 as fhn  # noqa: E402
from paper_2102_10340_b200.slab import SlabStepper  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
reps = 4
sim = fhn.Simulator(n, n)
sim.init(2, 42)
slabs = {}
for exact in (True, False):
    s = SlabStepper(n, n, rank=0, world=1, ghost=4, device=0, exact_blowup=exact)
    s.init(2, 42)
    s.fill_ghosts()
    slabs[exact] = s
for h in (sim,):
    h.advance(iters)
for s in slabs.values():
    s.advance(iters)
res = {"periodic": [], "slab+tee": [], "slab": []}
for _ in range(reps):
    sim.advance(iters)
    res["periodic"].append(sim.elapsed_ms())
    for exact, s in slabs.items():
        s.advance(iters)
        res["slab+tee" if exact else "slab"].append(s.elapsed_ms())
for k, v in res.items():
    best = min(v)
    print(f"{k:10s} {n}^2 x {iters}: min {best:.2f} ms  ({n * n * iters / best / 1e3:,.0f} Mcells/s)  all {['%.2f' % x for x in v]}")
