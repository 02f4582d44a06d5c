"""Generates tests/golden/golden.json from the REFERENCE ITSELF.

Runs the reference's own headers (oracle/_ref/librdcnn_ref.so, compiled
read-only from /root/reference/proj/include by oracle/Makefile) through its
public API -- init_center_square / init_full_random, run_timed on the
"reference" backend (engine.hpp:98-106), checksum (grid.hpp:101-116) -- and
records the digests.  The JSON travels to the GPU box; /root/reference does
not.  Re-run here with:  python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import DEFAULT_GENE7, Reference  # noqa: E402

SLOW_GROWTH = [0.1, -0.05, 1.3, -0.1, 1.0, 0.06, 1.0]   # a = -0.05
BLOWUP = [100.0, -0.3, 1.3, -0.1, 1.0, 0.06, 1.0]       # dt = 100 (test_engine.cpp:82-95)
PURE_DIFFUSION = [0.5, 0.0, 0.0, 0.0, 0.0, 0.1, 0.1]     # eps=0, c=0: diffusion-dominated

CASES = [
    # (name, rows, cols, typ, seed, gene7, iters)
    ("kat_crit1_256_typ1_s42_1000", 256, 256, 1, 42, DEFAULT_GENE7, 1000),   # test_output.txt:8
    ("kat_crit10_64_typ1_s42_200", 64, 64, 1, 42, DEFAULT_GENE7, 200),       # test_output.txt:23
    ("kat_blowup_16_dt100", 16, 16, 1, 42, BLOWUP, 1000),                    # test_engine.cpp:95
    ("blowup_32_dt100", 32, 32, 1, 42, BLOWUP, 1000),                        # acceptance 11 shape
    ("rand_32x48_s1001_25", 32, 48, 2, 1001, DEFAULT_GENE7, 25),             # test_kernels.cpp:141-157
    ("rand_17x23_s91_20", 17, 23, 2, 91, DEFAULT_GENE7, 20),                 # test_kernels.cpp:201-213
    ("rand_3x3_s5_50", 3, 3, 2, 5, DEFAULT_GENE7, 50),                       # minimum lattice
    ("rand_5x7_s6_33", 5, 7, 2, 6, DEFAULT_GENE7, 33),
    ("rand_24x36_s555_20", 24, 36, 2, 555, DEFAULT_GENE7, 20),               # test_kernels.cpp:187-199
    ("rand_128_s7_500", 128, 128, 2, 7, DEFAULT_GENE7, 500),                 # acceptance 2 shape
    ("rand_128_s11_10", 128, 128, 2, 11, DEFAULT_GENE7, 10),                 # acceptance 3 shape
    ("rand_100x260_s3_37", 100, 260, 2, 3, DEFAULT_GENE7, 37),
    ("rand_64x132_s4_41", 64, 132, 2, 4, DEFAULT_GENE7, 41),
    ("rand_512_s42_200", 512, 512, 2, 42, DEFAULT_GENE7, 200),               # FMA-drift case
    ("slow_512_typ1_s42_3000", 512, 512, 1, 42, SLOW_GROWTH, 3000),
    ("slow_300x200_typ1_s9_1111", 300, 200, 1, 9, SLOW_GROWTH, 1111),
    ("diffusion_40x40_s17_50", 40, 40, 2, 17, PURE_DIFFUSION, 50),
    ("rand_16_s8_dt0", 16, 16, 2, 8, [0.0, -0.3, 1.3, -0.1, 1.0, 0.06, 1.0], 3),  # test_kernels.cpp:83-96
]


CASES_F64 = [
    ("f64_rand_32x48_s1001_25", 32, 48, 2, 1001, DEFAULT_GENE7, 25),          # test_kernels.cpp:152-156
    ("f64_kat_256_typ1_s42_1000", 256, 256, 1, 42, DEFAULT_GENE7, 1000),
    ("f64_rand_17x23_s91_20", 17, 23, 2, 91, DEFAULT_GENE7, 20),
    ("f64_rand_128_s11_10", 128, 128, 2, 11, DEFAULT_GENE7, 10),              # acceptance 3 (double)
    ("f64_slow_300x200_typ1_s9_777", 300, 200, 1, 9, SLOW_GROWTH, 777),
    ("f64_blowup_16_dt100", 16, 16, 1, 42, BLOWUP, 1000),
]


# sweep_grid specs (sweep.hpp:255-326); the labels CSV is the golden output.
SWEEPS = [
    dict(x_param="du", xs=[0.02, 0.3], y_param="dv", ys=[0.5, 1.0, 5.0], nn=32, nm=32, iter_max=200, nssp=5),
    dict(x_param="du", xs=[0.3, 0.5, 0.7], y_param="dv", ys=[0.8, 1.0], nn=64, nm=64, iter_max=2000, nssp=5),
    dict(x_param="a", xs=[-0.3, -0.05], y_param="eps", ys=[-0.1, -0.05], typ=2, nn=40, nm=48, iter_max=100,
         nssp=4, seed=7, per_cell_seed=True),
    dict(x_param="a", xs=[-0.05, -0.3], y_param="c", ys=[1.0], nn=128, nm=128, iter_max=3000, nssp=5),
]


def main():
    ref = Reference()
    out = []
    for name, rows, cols, typ, seed, gene, iters in CASES:
        u, v = ref.init(typ, rows, cols, seed)
        init_ck = ref.checksum(rows, cols, u, v)
        fu, fv, bad, _ = ref.run_timed(rows, cols, u, v, iters, gene, backend="reference")
        ck = ref.checksum(rows, cols, fu, fv)
        out.append(dict(name=name, rows=rows, cols=cols, typ=typ, seed=seed, gene7=list(gene),
                        iters=iters, init_checksum=f"{init_ck:016x}", checksum=f"{ck:016x}",
                        bad_iter=bad, finite=bool(np.isfinite(fu).all() and np.isfinite(fv).all())))
        print(name, out[-1]["checksum"], bad)
    out64 = []
    for name, rows, cols, typ, seed, gene, iters in CASES_F64:
        u, v = ref.init_f64(typ, rows, cols, seed)
        init_ck = ref.checksum(rows, cols, u, v)
        fu, fv, bad, _ = ref.run_timed_f64(rows, cols, u, v, iters, gene, backend="reference")
        ck = ref.checksum(rows, cols, fu, fv)
        out64.append(dict(name=name, rows=rows, cols=cols, typ=typ, seed=seed, gene7=list(gene),
                          iters=iters, init_checksum=f"{init_ck:016x}", checksum=f"{ck:016x}",
                          bad_iter=bad, precision="double"))
        print(name, out64[-1]["checksum"], bad)
    sweeps = []
    for spec in SWEEPS:
        csv = ref.sweep_labels(**spec)
        sweeps.append(dict(spec=spec, labels_csv=csv))
        print("sweep", spec["x_param"], spec["y_param"], csv.count("\n") - 1, "cells")
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py via oracle/_ref (reference headers)",
                   "cases": out, "cases_f64": out64, "sweeps": sweeps}, f, indent=1)


if __name__ == "__main__":
    main()
