"""Golden outputs of the BASELINE.json configs at FULL size, from the REFERENCE
ITSELF (oracle/_ref: the reference headers compiled read-only, run through
their public API on this container's CPU cores).  Writes
tests/golden/baseline_golden.json; tests/test_baseline_gpu.py reproduces every
entry on the B200 bit for bit.  On 8 cores:

    python tests/golden/make_baseline_golden.py            # everything (~45 min)
    python tests/golden/make_baseline_golden.py cfg2_f64   # adds the fp64 entry (~1 min)

cfg1  256^2 typ=1 seed 42, default gene, 1000 iterations            (also a KAT)
cfg2  4096^2 typ=1 seed 42, slow-growth gene a=-0.05, 100 000 iterations,
      checksums every 10 000 (run_timed on the parallel backend)
cfg3  8192^2 synthetic 8-bit image (tools/cfg3_edge.py pattern, written by the
      reference's own PGM writer), typ=3 ka=1, default gene, 200 iterations
cfg4  sweep_grid du x dv = linspace(0.02,0.70,64) x linspace(0.50,1.20,64),
      128^2 typ=1 seed 42, 5000 iterations, nssp 5: the labels CSV
cfg5  32768^2 typ=2 seed 42, default gene, 100 iterations
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import DEFAULT_GENE7, Reference  # noqa: E402

SLOW_GROWTH = [0.1, -0.05, 1.3, -0.1, 1.0, 0.06, 1.0]


def cfg3_pixels(n: int) -> np.ndarray:
    """SURVEY §8d cfg3 pattern: checker blocks 37x53 (0.2/0.8) + 0.1 sin(0.05 i), 8-bit."""
    i = np.arange(n)[:, None]
    j = np.arange(n)[None, :]
    x = np.where(((i // 37) + (j // 53)) % 2 == 1, 0.8, 0.2) + 0.1 * np.sin(0.05 * i)
    return np.clip(np.round(x * 255), 0, 255).astype(np.uint8)


def cfg4_axes():
    return (list(np.linspace(0.02, 0.70, 64)), list(np.linspace(0.50, 1.20, 64)))


def main():
    ref = Reference()
    out = {"generator": "tests/golden/make_baseline_golden.py", "threads": ref.max_threads()}
    t0 = time.time()

    # cfg1
    u, v = ref.init(1, 256, 256, 42)
    u, v, bad, _ = ref.run_timed(256, 256, u, v, 1000, DEFAULT_GENE7, backend="parallel")
    out["cfg1"] = {"rows": 256, "cols": 256, "typ": 1, "seed": 42, "gene7": DEFAULT_GENE7, "iters": 1000,
                   "checksum": f"{ref.checksum(256, 256, u, v):016x}"}
    print("cfg1", out["cfg1"]["checksum"], f"{time.time() - t0:.0f}s", flush=True)

    # cfg3
    n = 8192
    from paper_2102_10340_b200 import imageio  # byte-identical PGM writer (tests/test_cli_io.py)
    img = os.path.join(ROOT, "tests", "golden", "_cfg3.pgm")
    imageio.write_pgm(img, cfg3_pixels(n))
    try:
        R, C, u, v = ref.init_image(img, 1.0)
    finally:
        os.remove(img)
    assert (R, C) == (n, n)
    init_sum = f"{ref.checksum(R, C, u, v):016x}"
    u, v, bad, _ = ref.run_timed(R, C, u, v, 200, DEFAULT_GENE7, backend="parallel")
    out["cfg3"] = {"rows": n, "cols": n, "typ": 3, "ka": 1.0, "gene7": DEFAULT_GENE7, "iters": 200,
                   "init_checksum": init_sum, "checksum": f"{ref.checksum(R, C, u, v):016x}", "bad_iter": bad}
    print("cfg3", out["cfg3"]["checksum"], f"{time.time() - t0:.0f}s", flush=True)
    del u, v

    # cfg5
    n = 32768
    u, v = ref.init(2, n, n, 42)
    init_sum = f"{ref.checksum(n, n, u, v):016x}"
    u, v, bad, _ = ref.run_timed(n, n, u, v, 100, DEFAULT_GENE7, backend="parallel")
    out["cfg5"] = {"rows": n, "cols": n, "typ": 2, "seed": 42, "gene7": DEFAULT_GENE7, "iters": 100,
                   "init_checksum": init_sum, "checksum": f"{ref.checksum(n, n, u, v):016x}", "bad_iter": bad}
    print("cfg5", out["cfg5"]["checksum"], f"{time.time() - t0:.0f}s", flush=True)
    del u, v

    # cfg4
    xs, ys = cfg4_axes()
    csv = ref.sweep_labels("du", xs, "dv", ys, nn=128, nm=128, iter_max=5000, nssp=5, seed=42,
                           parallel_cells=True)
    out["cfg4"] = {"x_param": "du", "xs": "linspace(0.02,0.70,64)", "y_param": "dv",
                   "ys": "linspace(0.50,1.20,64)", "rows": 128, "cols": 128, "typ": 1, "seed": 42,
                   "iter_max": 5000, "nssp": 5, "labels_csv_sha256": hashlib.sha256(csv.encode()).hexdigest(),
                   "labels_csv_lines": csv.count("\n")}
    with open(os.path.join(ROOT, "tests", "golden", "cfg4_labels.csv"), "w") as f:
        f.write(csv)
    print("cfg4", out["cfg4"]["labels_csv_sha256"][:16], f"{time.time() - t0:.0f}s", flush=True)

    # cfg2 (the long one)
    n = 4096
    u, v = ref.init(1, n, n, 42)
    sums = []
    for k in range(10):
        u, v, bad, _ = ref.run_timed(n, n, u, v, 10000, SLOW_GROWTH, backend="parallel")
        assert bad == 0
        sums.append(f"{ref.checksum(n, n, u, v):016x}")
        print("cfg2", (k + 1) * 10000, sums[-1], f"{time.time() - t0:.0f}s", flush=True)
    out["cfg2"] = {"rows": n, "cols": n, "typ": 1, "seed": 42, "gene7": SLOW_GROWTH, "iters": 100000,
                   "checksums_every_10000": sums}

    out["seconds"] = round(time.time() - t0, 1)
    with open(os.path.join(ROOT, "tests", "golden", "baseline_golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("done", out["seconds"], "s")


def add_cfg2_f64():
    """fp64 (the reference's double instantiation) on the cfg2 lattice: the
    first 1000 iterations, merged into the existing JSON (~1 minute)."""
    ref = Reference()
    path = os.path.join(ROOT, "tests", "golden", "baseline_golden.json")
    with open(path) as f:
        out = json.load(f)
    n = 4096
    u, v = ref.init_f64(1, n, n, 42)
    u, v, bad, _ = ref.run_timed_f64(n, n, u, v, 1000, SLOW_GROWTH, backend="parallel")
    out["cfg2_f64"] = {"rows": n, "cols": n, "typ": 1, "seed": 42, "gene7": SLOW_GROWTH, "iters": 1000,
                       "checksum": f"{ref.checksum(n, n, u, v):016x}", "bad_iter": bad}
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("cfg2_f64", out["cfg2_f64"]["checksum"])


if __name__ == "__main__":
    if sys.argv[1:] == ["cfg2_f64"]:
        add_cfg2_f64()
    else:
        main()
