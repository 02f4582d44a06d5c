"""ctypes wrappers of the test-only CPU checkers (TEST INFRASTRUCTURE ONLY).

* :class:`Oracle`    -- oracle/liboracle.so, the C restatement (fhn_oracle.c)
* :class:`Reference` -- oracle/_ref/librdcnn_ref.so, the reference's own
                        headers compiled read-only (ref_driver.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only to check or time the CPU path.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import c_double, c_int, c_long, c_size_t, c_uint32, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "librdcnn_ref.so")

DEFAULT_GENE7 = [0.1, -0.3, 1.3, -0.1, 1.0, 0.06, 1.0]  # dt,a,b,eps,c,Du,Dv (gene.hpp:13-24)


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _p(a: np.ndarray):
    return c_void_p(a.ctypes.data)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.orc_run_f32.restype = c_long
        L.orc_run_f32.argtypes = [c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_long]
        L.orc_run_f64.restype = c_long
        L.orc_run_f64.argtypes = L.orc_run_f32.argtypes
        L.orc_step_f32.restype = c_int
        L.orc_step_f32.argtypes = [c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
        L.orc_checksum.restype = c_uint64
        L.orc_checksum.argtypes = [c_void_p, c_void_p, c_size_t]
        L.orc_params_f32.argtypes = [c_void_p, c_void_p]
        L.orc_init_center_square_f32.restype = c_int
        L.orc_init_center_square_f32.argtypes = [c_int, c_int, c_uint64, c_void_p, c_void_p]
        L.orc_init_full_random_f32.argtypes = [c_int, c_int, c_uint64, c_void_p, c_void_p]
        L.orc_init_from_image_f32.argtypes = [c_void_p, c_size_t, c_double, c_void_p, c_void_p]
        for n in ("orc_reaction_u_f32", "orc_reaction_v_f32"):
            getattr(L, n).restype = ctypes.c_float
            getattr(L, n).argtypes = [ctypes.c_float, ctypes.c_float, c_void_p]
        for n in ("orc_reaction_u_f64", "orc_reaction_v_f64"):
            getattr(L, n).restype = c_double
            getattr(L, n).argtypes = [c_double, c_double, c_void_p]
        L.orc_cell_update_f64.argtypes = [c_double] * 4 + [c_void_p, c_void_p, c_void_p]
        L.orc_laplacian5_f64.restype = c_double
        L.orc_laplacian5_f64.argtypes = [c_void_p, c_int, c_int, c_int, c_int]
        L.div3_sweep.restype = c_uint64
        L.div3_sweep.argtypes = [c_uint64, c_uint64, ctypes.POINTER(c_uint32)]
        L.div3_two_op_sweep.restype = c_uint64
        L.div3_two_op_sweep.argtypes = [c_int, ctypes.POINTER(c_uint32), ctypes.POINTER(c_uint32)]
        self.L = L

    def params(self, gene7=DEFAULT_GENE7) -> np.ndarray:
        g = np.asarray(gene7, np.float64)
        p = np.zeros(7, np.float32)
        self.L.orc_params_f32(_p(g), _p(p))
        return p

    def init(self, typ: int, rows: int, cols: int, seed: int):
        u = np.zeros(rows * cols, np.float32)
        v = np.zeros(rows * cols, np.float32)
        if typ == 1:
            if self.L.orc_init_center_square_f32(rows, cols, seed, _p(u), _p(v)) != 0:
                raise ValueError("grid too small for typ=1")
        else:
            self.L.orc_init_full_random_f32(rows, cols, seed, _p(u), _p(v))
        return u, v

    def init_image(self, px: np.ndarray, ka: float = 1.0):
        px = np.ascontiguousarray(px, np.uint8).reshape(-1)
        u = np.zeros(px.size, np.float32)
        v = np.zeros(px.size, np.float32)
        self.L.orc_init_from_image_f32(_p(px), px.size, ka, _p(u), _p(v))
        return u, v

    def run(self, rows: int, cols: int, u: np.ndarray, v: np.ndarray, iters: int, gene7=DEFAULT_GENE7):
        """Returns (u, v, bad_iter) after iters steps (stops at the first non-finite)."""
        u = np.array(u, np.float32, copy=True).reshape(-1)
        v = np.array(v, np.float32, copy=True).reshape(-1)
        su = np.empty_like(u)
        sv = np.empty_like(v)
        p = self.params(gene7)
        bad = self.L.orc_run_f32(rows, cols, _p(u), _p(v), _p(su), _p(sv), _p(p), iters)
        return u, v, int(bad)

    def checksum(self, u: np.ndarray, v: np.ndarray) -> int:
        u = np.ascontiguousarray(u)
        v = np.ascontiguousarray(v)
        return int(self.L.orc_checksum(_p(u), _p(v), u.nbytes))

    # ---- fp64 (the reference templates instantiate double as well) --------
    def init_f64(self, typ: int, rows: int, cols: int, seed: int):
        u = np.zeros(rows * cols, np.float64)
        v = np.zeros(rows * cols, np.float64)
        if typ == 1:
            self.L.orc_init_center_square_f64.argtypes = [c_int, c_int, c_uint64, c_void_p, c_void_p]
            if self.L.orc_init_center_square_f64(rows, cols, seed, _p(u), _p(v)) != 0:
                raise ValueError("grid too small for typ=1")
        else:
            self.L.orc_init_full_random_f64.argtypes = [c_int, c_int, c_uint64, c_void_p, c_void_p]
            self.L.orc_init_full_random_f64(rows, cols, seed, _p(u), _p(v))
        return u, v

    def run_f64(self, rows: int, cols: int, u, v, iters: int, gene7=DEFAULT_GENE7):
        u = np.array(u, np.float64, copy=True).reshape(-1)
        v = np.array(v, np.float64, copy=True).reshape(-1)
        su = np.empty_like(u)
        sv = np.empty_like(v)
        p = np.asarray(gene7, np.float64)  # make_params<double>: no narrowing
        bad = self.L.orc_run_f64(rows, cols, _p(u), _p(v), _p(su), _p(sv), _p(p), iters)
        return u, v, int(bad)

    def div3_sweep(self, lo: int = 0, hi: int = 1 << 32):
        first = c_uint32(0)
        n = self.L.div3_sweep(lo, hi, ctypes.byref(first))
        return int(n), int(first.value)

    def div3_two_op_sweep(self, mode: int):
        """(mismatches, smallest, largest bad pattern) of the gated 2-op x/3
        over every x >= +0: mode 0 the raw quotient, mode 1 RN(c - x/3)."""
        lo, hi = c_uint32(0), c_uint32(0)
        n = self.L.div3_two_op_sweep(mode, ctypes.byref(lo), ctypes.byref(hi))
        return int(n), int(lo.value), int(hi.value)


class Reference:
    """The reference's own code path (engine.hpp run/run_timed on its backends)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (reference tree was not available to build it)")
        L = ctypes.CDLL(path)
        L.ref_init_f32.restype = c_int
        L.ref_init_f32.argtypes = [c_int, c_int, c_int, c_uint64, c_void_p, c_void_p]
        L.ref_run_timed_f32.restype = c_int
        L.ref_run_timed_f32.argtypes = [c_int, c_int, c_void_p, c_void_p, c_void_p, ctypes.c_char_p,
                                        c_int, c_long, ctypes.POINTER(c_long), ctypes.POINTER(c_double)]
        L.ref_run_f32.restype = c_int
        L.ref_run_f32.argtypes = [c_int, c_int, c_void_p, c_void_p, c_void_p, ctypes.c_char_p, c_long,
                                  c_int, c_void_p, c_void_p, c_void_p, ctypes.POINTER(c_long)]
        L.ref_checksum_f32.restype = c_uint64
        L.ref_checksum_f32.argtypes = [c_int, c_int, c_void_p, c_void_p]
        L.ref_max_threads.restype = c_int
        self.L = L

    def max_threads(self) -> int:
        return int(self.L.ref_max_threads())

    def set_threads(self, n: int) -> None:
        """OpenMP threads for the reference's regions without an explicit count
        (the parallel_cells sweep loop); torchrun presets OMP_NUM_THREADS=1."""
        self.L.ref_set_threads(int(n))

    def init(self, typ: int, rows: int, cols: int, seed: int):
        u = np.zeros(rows * cols, np.float32)
        v = np.zeros(rows * cols, np.float32)
        if self.L.ref_init_f32(typ, rows, cols, seed, _p(u), _p(v)) != 0:
            raise ValueError("reference init rejected the shape")
        return u, v

    def run_timed(self, rows, cols, u, v, iters, gene7=DEFAULT_GENE7, ka=1.0, backend="parallel",
                  threads=0):
        """Returns (u, v, bad_iter, seconds) via the reference run_timed."""
        u = np.array(u, np.float32, copy=True).reshape(-1)
        v = np.array(v, np.float32, copy=True).reshape(-1)
        g8 = np.asarray(list(gene7) + [ka], np.float64)
        bad = c_long(0)
        sec = c_double(0)
        rc = self.L.ref_run_timed_f32(rows, cols, _p(u), _p(v), _p(g8), backend.encode(), threads, iters,
                                      ctypes.byref(bad), ctypes.byref(sec))
        if rc == 1:
            raise ValueError("reference rejected the arguments")
        return u, v, int(bad.value), float(sec.value)

    def run(self, rows, cols, u, v, iter_max, nssp, gene7=DEFAULT_GENE7, backend="reference"):
        """engine.hpp run(): returns (frames_u, frames_v, labels, rc, bad_iter)."""
        n = rows * cols
        fu = np.zeros((nssp + 1) * n, np.float32)
        fv = np.zeros((nssp + 1) * n, np.float32)
        labels = np.zeros(nssp + 1, np.int64)
        bad = c_long(0)
        g8 = np.asarray(list(gene7) + [1.0], np.float64)
        u = np.ascontiguousarray(u, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        rc = self.L.ref_run_f32(rows, cols, _p(u), _p(v), _p(g8), backend.encode(), iter_max, nssp,
                                _p(fu), _p(fv), _p(labels), ctypes.byref(bad))
        return fu.reshape(nssp + 1, n), fv.reshape(nssp + 1, n), labels, rc, int(bad.value)

    def checksum(self, rows, cols, u, v) -> int:
        if np.asarray(u).dtype == np.float64:
            f = self.L.ref_checksum_f64
            f.restype = c_uint64
            f.argtypes = [c_int, c_int, c_void_p, c_void_p]
            return int(f(rows, cols, _p(np.ascontiguousarray(u)), _p(np.ascontiguousarray(v))))
        return int(self.L.ref_checksum_f32(rows, cols, _p(np.ascontiguousarray(u)), _p(np.ascontiguousarray(v))))

    def sweep_labels(self, x_param, xs, y_param, ys, gene7=DEFAULT_GENE7, ka=1.0, typ=1, nn=32, nm=32,
                     iter_max=100, nssp=5, seed=42, per_cell_seed=False, parallel_cells=False) -> str:
        """The reference's sweep_grid labels CSV (sweep.hpp:227-247)."""
        f = self.L.ref_sweep_labels_par_f32 if parallel_cells else self.L.ref_sweep_labels_f32
        f.restype = c_int
        f.argtypes = [ctypes.c_char_p, c_void_p, c_int, ctypes.c_char_p, c_void_p, c_int, c_void_p, c_int,
                      c_int, c_int, c_long, c_int, c_uint64, c_int, ctypes.c_char_p, c_size_t]
        xa = np.asarray(xs, np.float64)
        ya = np.asarray(ys, np.float64)
        g8 = np.asarray(list(gene7) + [ka], np.float64)
        buf = ctypes.create_string_buffer(1 << 22)
        rc = f(x_param.encode(), _p(xa), len(xa), y_param.encode(), _p(ya), len(ya), _p(g8), typ, nn, nm,
               iter_max, nssp, seed, int(per_cell_seed), buf, len(buf))
        if rc != 0:
            raise ValueError("reference sweep_grid rejected the spec")
        return buf.value.decode()

    def init_image(self, path: str, ka: float = 1.0):
        """The reference's typ=3 state from an image file (load_grayscale +
        init_from_image); returns (rows, cols, u, v)."""
        f = self.L.ref_init_image_f32
        f.restype = c_int
        f.argtypes = [ctypes.c_char_p, c_double, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t]
        r, c = ctypes.c_int(), ctypes.c_int()
        cap = 1 << 27
        u = np.empty(cap, np.float32)
        v = np.empty(cap, np.float32)
        rc = f(path.encode(), ka, ctypes.byref(r), ctypes.byref(c), _p(u), _p(v), cap)
        if rc != 0:
            raise ValueError(f"reference could not load {path} (rc {rc})")
        n = r.value * c.value
        return r.value, c.value, u[:n].copy(), v[:n].copy()

    def format_double(self, x: float) -> str:
        f = self.L.ref_format_double
        f.restype = c_int
        f.argtypes = [c_double, ctypes.c_char_p, c_size_t]
        buf = ctypes.create_string_buffer(64)
        f(x, buf, 64)
        return buf.value.decode()

    def init_f64(self, typ: int, rows: int, cols: int, seed: int):
        u = np.zeros(rows * cols, np.float64)
        v = np.zeros(rows * cols, np.float64)
        f = self.L.ref_init_f64
        f.restype = c_int
        f.argtypes = [c_int, c_int, c_int, c_uint64, c_void_p, c_void_p]
        if f(typ, rows, cols, seed, _p(u), _p(v)) != 0:
            raise ValueError("reference init rejected the shape")
        return u, v

    def run_timed_f64(self, rows, cols, u, v, iters, gene7=DEFAULT_GENE7, ka=1.0, backend="parallel",
                      threads=0):
        u = np.array(u, np.float64, copy=True).reshape(-1)
        v = np.array(v, np.float64, copy=True).reshape(-1)
        g8 = np.asarray(list(gene7) + [ka], np.float64)
        bad = c_long(0)
        sec = c_double(0)
        f = self.L.ref_run_timed_f64
        f.restype = c_int
        f.argtypes = self.L.ref_run_timed_f32.argtypes
        rc = f(rows, cols, _p(u), _p(v), _p(g8), backend.encode(), threads, iters, ctypes.byref(bad),
               ctypes.byref(sec))
        if rc == 1:
            raise ValueError("reference rejected the arguments")
        return u, v, int(bad.value), float(sec.value)
