import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2102_10340_b200 as fhn
B = 4096
st = fhn.init_center_square(128, 128, 42)
u_in = torch.empty(B, 128 * 128, dtype=torch.float32).pin_memory(); u_in[:] = torch.from_numpy(st.u)
v_in = torch.empty(B, 128 * 128, dtype=torch.float32).pin_memory(); v_in[:] = torch.from_numpy(st.v)
with fhn.Simulator(128, 128, batch=B, levels=4) as sim:
    for mode in ("init", "upload", "init", "upload"):
        if mode == "init": sim.init(1, 42)
        else: sim.upload(u_in.numpy(), v_in.numpy())
        torch.cuda.synchronize()
        for adv in (0, 1000):
            if adv: sim.advance(adv)
            t = time.perf_counter(); d = sim.checksums(); t1 = time.perf_counter() - t
            t = time.perf_counter(); d = sim.checksums(); t2 = time.perf_counter() - t
            print(f"{mode} adv={adv}: checksums {t1*1e3:.1f} ms then {t2*1e3:.1f} ms  digest0 {int(d[0]):016x}", flush=True)
