"""ctypes binding of the C-ABI in include/rdcnn_cuda.h.

The shared library is built in-tree by ``__graft_entry__.build()``
(``paper_2102_10340_b200/librdcnn_cuda.so``).  There is no fallback: if the
library is missing, importing :mod:`paper_2102_10340_b200` still works (so the
CPU-only test suite can inspect it), but every compute entry point raises
:class:`LibraryMissing`.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_long, c_size_t, c_uint, c_uint32, c_uint64, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
# RDCNN_LIB: load another build of the extension (A/B measurements only).
LIB_PATH = os.environ.get("RDCNN_LIB") or os.path.join(HERE, "librdcnn_cuda.so")

RDCNN_OK, RDCNN_EINVAL, RDCNN_EBLOWUP, RDCNN_ECUDA = 0, 1, 2, 3
RDCNN_STRICT, RDCNN_FAST = 0, 1


class LibraryMissing(RuntimeError):
    """The CUDA extension was not built; run __graft_entry__.build()."""


class ParamsF32(ctypes.Structure):
    """rdcnn_params_f32: gene narrowed to fp32 in kernel order (gene.hpp:39-41)."""

    _fields_ = [(n, c_float) for n in ("dt", "a", "b", "eps", "c", "du", "dv")]


class ParamsF64(ctypes.Structure):
    """rdcnn_params_f64: the gene in fp64, kernel order."""

    _fields_ = [(n, c_double) for n in ("dt", "a", "b", "eps", "c", "du", "dv")]


class PeerDesc(ctypes.Structure):
    """rdcnn_slab_peer_desc: one slab's exported peer memory (IPC handles +
    in-process pointers) for the fused peer ring."""

    _fields_ = [("ipc", (ctypes.c_uint8 * 64) * 3), ("ptr", c_uint64 * 3), ("pid", ctypes.c_int64),
                ("device", ctypes.c_int32), ("rows", ctypes.c_int32), ("cols", ctypes.c_int32),
                ("ghost", ctypes.c_int32), ("ipc_ok", ctypes.c_int32)]


# name -> (restype, argtypes); exactly the symbols include/rdcnn_cuda.h declares.
SIGNATURES = {
    "rdcnn_abi_version": (c_int, []),
    "rdcnn_last_error": (c_char_p, []),
    "rdcnn_device_count": (c_int, [POINTER(c_int)]),
    "rdcnn_params_from_gene": (None, [POINTER(c_double), POINTER(ParamsF32)]),
    "rdcnn_sim_create": (c_int, [c_int, c_int, c_int, c_int, c_int, POINTER(c_void_p)]),
    "rdcnn_sim_create_f64": (c_int, [c_int, c_int, c_int, c_int, POINTER(c_void_p)]),
    "rdcnn_sim_precision": (c_int, [c_void_p, POINTER(c_int)]),
    "rdcnn_sim_destroy": (None, [c_void_p]),
    "rdcnn_sim_set_params_f64": (c_int, [c_void_p, POINTER(ParamsF64), c_int]),
    "rdcnn_sim_upload_f64": (c_int, [c_void_p, c_void_p, c_void_p]),
    "rdcnn_sim_download_f64": (c_int, [c_void_p, c_void_p, c_void_p]),
    "rdcnn_init_center_square_host_f64": (c_int, [c_int, c_int, c_uint64, c_void_p, c_void_p]),
    "rdcnn_init_full_random_host_f64": (c_int, [c_int, c_int, c_uint64, c_void_p, c_void_p]),
    "rdcnn_checksum_f64": (c_uint64, [c_void_p, c_void_p, c_size_t]),
    "rdcnn_selftest_div3_f64": (c_int, [c_int, c_uint64, POINTER(c_uint64), POINTER(c_uint64)]),
    "rdcnn_sim_set_params": (c_int, [c_void_p, POINTER(ParamsF32), c_int]),
    "rdcnn_sim_upload": (c_int, [c_void_p, c_void_p, c_void_p]),
    "rdcnn_sim_download": (c_int, [c_void_p, c_void_p, c_void_p]),
    "rdcnn_sim_init": (c_int, [c_void_p, c_int, c_uint64]),
    "rdcnn_sim_init_image": (c_int, [c_void_p, c_void_p, c_double]),
    "rdcnn_sim_advance": (c_int, [c_void_p, c_long, POINTER(c_long)]),
    "rdcnn_sim_elapsed_ms": (c_int, [c_void_p, POINTER(c_double)]),
    "rdcnn_sim_launch_count": (c_int, [c_void_p, POINTER(c_long)]),
    "rdcnn_sim_set_tuning": (c_int, [c_void_p, c_int, c_int]),
    "rdcnn_sim_set_persistent": (c_int, [c_void_p, c_int]),
    "rdcnn_sim_trace_launch": (c_int, [c_void_p, c_int, c_void_p, ctypes.c_longlong,
                                       POINTER(ctypes.c_longlong)]),
    "rdcnn_sim_stream": (c_int, [c_void_p, POINTER(c_void_p)]),
    "rdcnn_sim_device_state": (c_int, [c_void_p, POINTER(c_void_p), POINTER(c_void_p)]),
    "rdcnn_slab_create": (c_int, [c_int, c_int, c_int, c_int, c_int, POINTER(c_void_p)]),
    "rdcnn_slab_init": (c_int, [c_void_p, c_int, c_uint64, c_int, c_int]),
    "rdcnn_slab_step_boundary": (c_int, [c_void_p, c_int, c_void_p]),
    "rdcnn_slab_step_interior": (c_int, [c_void_p, c_int, c_void_p]),
    "rdcnn_slab_swap": (c_int, [c_void_p]),
    "rdcnn_slab_rows_ptr": (c_int, [c_void_p, c_int, POINTER(c_void_p), POINTER(c_void_p)]),
    "rdcnn_slab_poll_blowup": (c_int, [c_void_p, POINTER(c_int), POINTER(c_uint)]),
    "rdcnn_nccl_unique_id": (c_int, [c_void_p]),
    "rdcnn_slab_attach_ring": (c_int, [c_void_p, c_void_p, c_int, c_int]),
    "rdcnn_slab_fill_ghosts": (c_int, [c_void_p]),
    "rdcnn_slab_advance": (c_int, [c_void_p, c_long, POINTER(c_long)]),
    "rdcnn_slab_peer_export": (c_int, [c_void_p, POINTER(PeerDesc)]),
    "rdcnn_slab_attach_peers": (c_int, [c_void_p, c_int, c_int, POINTER(PeerDesc), POINTER(PeerDesc)]),
    "rdcnn_slab_step_fused": (c_int, [c_void_p, c_int, c_void_p]),
    "rdcnn_slab_checkpoint_enable": (c_int, [c_void_p, c_int]),
    "rdcnn_slab_restore": (c_int, [c_void_p]),
    "rdcnn_slab_checkpoint_age": (c_int, [c_void_p, POINTER(c_long)]),
    "rdcnn_ring_create": (c_int, [c_int, c_int, POINTER(c_int), c_int, c_int, c_int, POINTER(c_void_p)]),
    "rdcnn_ring_destroy": (None, [c_void_p]),
    "rdcnn_ring_slab": (c_int, [c_void_p, c_int, POINTER(c_void_p), POINTER(c_int), POINTER(c_int),
                                POINTER(c_int)]),
    "rdcnn_ring_set_params": (c_int, [c_void_p, POINTER(ParamsF32)]),
    "rdcnn_ring_set_levels": (c_int, [c_void_p, c_int]),
    "rdcnn_ring_set_exact": (c_int, [c_void_p, c_int]),
    "rdcnn_ring_init": (c_int, [c_void_p, c_int, c_uint64]),
    "rdcnn_ring_upload": (c_int, [c_void_p, c_void_p, c_void_p]),
    "rdcnn_ring_download": (c_int, [c_void_p, c_void_p, c_void_p]),
    "rdcnn_ring_advance": (c_int, [c_void_p, c_long, POINTER(c_long)]),
    "rdcnn_ring_elapsed_ms": (c_int, [c_void_p, POINTER(c_double)]),
    "rdcnn_ring_launch_count": (c_int, [c_void_p, POINTER(c_long)]),
    "rdcnn_ring_trace_block": (c_int, [c_void_p, c_int, c_void_p, ctypes.c_longlong,
                                       POINTER(ctypes.c_longlong)]),
    "rdcnn_sim_checksums": (c_int, [c_void_p, c_void_p]),
    "rdcnn_sim_frames_reserve": (c_int, [c_void_p, c_int]),
    "rdcnn_sim_frame_capture": (c_int, [c_void_p, c_int]),
    "rdcnn_sim_frame_download": (c_int, [c_void_p, c_int, c_void_p]),
    "rdcnn_sim_frame_stats": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "rdcnn_sim_frame_active": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "rdcnn_sim_frame_normalize": (c_int, [c_void_p, c_int, c_int, c_double, c_double, c_void_p]),
    "rdcnn_sim_frame_normalize_auto": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "rdcnn_init_center_square_host": (c_int, [c_int, c_int, c_uint64, c_void_p, c_void_p]),
    "rdcnn_init_full_random_host": (c_int, [c_int, c_int, c_uint64, c_void_p, c_void_p]),
    "rdcnn_checksum_f32": (c_uint64, [c_void_p, c_void_p, c_size_t]),
    "rdcnn_selftest_div3": (c_int, [c_int, c_int, POINTER(c_uint64), POINTER(c_uint32)]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and return the CUDA extension; raise LibraryMissing if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LibraryMissing(
            f"{path} not found: build the CUDA extension with "
            "`python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class RdcnnError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def last_error() -> str:
    msg = load().rdcnn_last_error()
    return msg.decode() if msg else ""


def check(code: int) -> int:
    if code == RDCNN_OK or code == RDCNN_EBLOWUP:
        return code
    raise RdcnnError(code, last_error())
