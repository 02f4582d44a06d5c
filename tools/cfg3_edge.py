"""cfg3 (BASELINE configs[2]): CNN edge detection on a synthetic 8192^2 image,
T = 200, nssp = 5, through the reference CLI front end (`simulate --typ 3`),
timed phase by phase.  The image is the SURVEY §8d pattern (piecewise-constant
blocks + a gradient, 8-bit), written as PGM first."""
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = __file__.rsplit("/tools/", 1)[0]
sys.path.insert(0, ROOT)
from paper_2102_10340_b200 import imageio  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
i = np.arange(n)[:, None]
j = np.arange(n)[None, :]
x = np.where(((i // 37) + (j // 53)) % 2 == 1, 0.8, 0.2) + 0.1 * np.sin(0.05 * i)
px = np.clip(np.round(x * 255), 0, 255).astype(np.uint8)
d = tempfile.mkdtemp()
img = os.path.join(d, "edges.pgm")
imageio.write_pgm(img, px)
t0 = time.perf_counter()
r = subprocess.run([sys.executable, "-m", "paper_2102_10340_b200", "simulate", "--typ", "3", "--image", img,
                    "--iters", "200", "--nssp", "5", "--out", os.path.join(d, "run")],
                   cwd=ROOT, capture_output=True, text=True)
wall = time.perf_counter() - t0
print(r.stdout[-1500:])
print(r.stderr[-800:])
print(f"cfg3 {n}^2 T=200 nssp=5 via CLI: wall {wall:.2f} s (incl. interpreter start, image I/O, PGM/PNG output); "
      f"cell-updates {n * n * 200:.3e}")
