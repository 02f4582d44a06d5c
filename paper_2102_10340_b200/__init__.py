"""B200-native FitzHugh-Nagumo RD-CNN time stepper (arXiv 2102.10340).

The hot path is hand-written sm_100a CUDA behind the C-ABI in
include/rdcnn_cuda.h; this package is its Python host side (a mirror of the
reference's C++ API, see :mod:`.engine`) plus the multi-GPU slab driver
(:mod:`.slab`).
"""
from ._lib import LIB_PATH, LibraryMissing, RdcnnError, last_error, load  # noqa: F401
from .engine import (  # noqa: F401
    Backend, BlowUpError, Gene, GridState, Pipeline, RunConfig, RunOutput, ScheduleError, Simulator,
    SnapshotBuffer, StepBuffers, checksum, checksum_hex, gene_valid, init_center_square,
    init_from_image, init_full_random, initial_state, make_backend, params_from_gene, run,
    run_timed, step, validate_config,
)
from .slab import Ring  # noqa: F401

__version__ = "0.1.0"
