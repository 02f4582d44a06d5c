import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2102_10340_b200 as fhn
from paper_2102_10340_b200.slab import SlabStepper
from oracle.oracle import Oracle
o = Oracle()
rows, cols = 64, 96
u0, v0 = o.init(2, rows, cols, 5)
for ghost in (2, 4, 8):
  for iters in (1, 2, 4, 5, 8, 9):
    ou, ov, _ = o.run(rows, cols, u0, v0, iters)
    s = SlabStepper(rows, cols, 0, 1, ghost=ghost, device=0)
    s.upload(u0, v0); s.fill_ghosts(); s.advance(iters); torch.cuda.synchronize()
    u, v = s.download()
    d = (u.view(np.uint32) != ou.view(np.uint32)).reshape(rows, cols)
    r = np.nonzero(d.any(1))[0]; c = np.nonzero(d.any(0))[0]
    print(ghost, iters, "bad rows", r[:20], "bad cols", c[:20], d.sum())
    s.close()
