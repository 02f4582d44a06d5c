import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2102_10340_b200 as fhn
for n, it in ((512, 20000), (1024, 10000), (2048, 8000), (4096, 4000)):
    with fhn.Simulator(n, n, levels=4, persistent=-1) as sim:
        sim.set_params(fhn.Gene(a=-0.05)); sim.init(1, 42)
        ts = []
        for _ in range(4):
            sim.advance(it); ts.append(sim.elapsed_ms())
        u, v = sim.download()
        print(f"{n}^2: {n*n*it/min(ts[1:])/1e3:,.0f} Mcells/s  checksum {fhn.checksum(fhn.GridState(n, n, u, v)):016x}", flush=True)
