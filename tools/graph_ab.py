"""Mid-size lattices with CUDA-graph replay on/off (RDCNN_GRAPH) at fusion depth K
(argv[1], default 4): the best of three same-length advances after a first one."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2102_10340_b200 as fhn

levels = int(sys.argv[1]) if len(sys.argv) > 1 else 4
for n, it in ((512, 20000), (1024, 10000), (2048, 8000), (4096, 4000)):
    with fhn.Simulator(n, n, levels=levels, persistent=-1) as sim:
        sim.set_params(fhn.Gene(a=-0.05)); sim.init(1, 42)
        ts = []
        for _ in range(4):
            sim.advance(it); ts.append(sim.elapsed_ms())
        u, v = sim.download()
        print(f"K={levels} {n}^2: {n*n*it/min(ts[1:])/1e3:,.0f} Mcells/s  checksum {fhn.checksum(fhn.GridState(n, n, u, v)):016x}", flush=True)
