"""Row-slab sharding of one large torus across GPUs.

Each rank owns ``rows // world`` consecutive rows of the global lattice
(SURVEY.md §8e); rank r-1 is above, r+1 below, and the ring is periodic
(rank 0's top ghosts are rank P-1's last rows: the torus row wrap of
kernels.hpp:46-47).  Column wrap stays inside each slab.  Two native
transports advance a block of ``k <= ghost`` time levels:

* ``p2p`` (default): ONE fused launch per block.  The warps whose level-0
  rows reach beyond the slab first acquire the neighbour's ready word, then
  stage those rows straight from the neighbour's INPUT buffer over peer
  memory (CUDA IPC mappings over NVLink; plain pointers in-process), and
  finally publish their own word with a release store ("my edge rows of
  this block are written, and I have finished reading yours").  Nothing is
  copied into ghost rows; interior warps never wait, so the exchange
  overlaps the step tile by tile.
* ``nccl``: boundary kernel -> NCCL send/recv of the edge rows into the
  ghost rows on a comm stream, overlapped with the interior kernel; wait;
  swap.

Two ways to run it:

* :class:`Ring` -- ONE process drives every slab (``rdcnn_ring_*`` in the
  C-ABI): one host thread per device, in-process peer pointers, the exact
  blow-up replay in native code.  ``bench.py --gpus N`` without torchrun.
* :class:`SlabStepper` -- one process per GPU (torchrun), descriptors
  shared through torch.distributed, CUDA IPC between the processes.

Arithmetic per cell is unchanged, so the result is bit-identical to the
single-GPU periodic run at any world size.

The Python-driven exchange is a plain function of four row blocks so it can
be exercised on CPU tensors with the gloo backend (tests/test_slab_gloo.py).
"""
from __future__ import annotations

import ctypes
from typing import Callable, Optional

from . import _lib
from ._lib import RDCNN_FAST, RDCNN_STRICT, check, load


class _CudaRows:
    """Zero-copy view of device rows for torch (``__cuda_array_interface__``)."""

    def __init__(self, ptr: int, rows: int, width: int):
        self.__cuda_array_interface__ = {
            "shape": (rows, width), "typestr": "<f4", "data": (int(ptr), False), "version": 2,
        }


class Ring:
    """One torus of ``global_rows x cols`` split into row slabs in THIS
    process (rdcnn_ring_*): slab r on ``devices[r]`` (entries may repeat),
    the fused peer halo exchange between them, one host thread per device,
    and the exact blow-up iteration.  Same surface as ``engine.Simulator``
    for one fp32 lattice (``advance`` returns ``first_bad[1]``)."""

    def __init__(self, global_rows: int, cols: int, devices, ghost: int = 4, mode: str = "strict",
                 levels: Optional[int] = None, exact: bool = True):
        self._lib = load()
        devs = [int(d) for d in devices]
        if not devs:
            raise ValueError("a ring needs at least one device")
        if mode not in ("strict", "fast"):
            raise ValueError(f"unknown mode {mode}")
        self.rows, self.cols, self.batch = int(global_rows), int(cols), 1
        self.devices, self.ghost, self.mode = devs, int(ghost), mode
        self.precision = "single"
        import numpy as np
        self.dtype = np.dtype(np.float32)
        arr = (ctypes.c_int * len(devs))(*devs)
        h = ctypes.c_void_p()
        check(self._lib.rdcnn_ring_create(self.rows, self.cols, arr, len(devs), self.ghost,
                                          RDCNN_FAST if mode == "fast" else RDCNN_STRICT, ctypes.byref(h)))
        self._h = h
        if levels is not None:
            self.set_levels(levels)
        check(self._lib.rdcnn_ring_set_exact(self._h, 1 if exact else 0))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.rdcnn_ring_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def slab(self, r: int):
        """(row_offset, rows, device) of slab r."""
        off, rows, dev = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        check(self._lib.rdcnn_ring_slab(self._h, int(r), None, ctypes.byref(off), ctypes.byref(rows),
                                        ctypes.byref(dev)))
        return off.value, rows.value, dev.value

    def set_levels(self, levels: int):
        check(self._lib.rdcnn_ring_set_levels(self._h, int(levels)))

    def set_params(self, gene):
        from .engine import params_from_gene
        p = gene if isinstance(gene, _lib.ParamsF32) else params_from_gene(gene)
        check(self._lib.rdcnn_ring_set_params(self._h, ctypes.byref(p)))

    def init(self, typ: int, seed: int):
        check(self._lib.rdcnn_ring_init(self._h, int(typ), ctypes.c_uint64(seed)))

    def upload(self, u, v):
        import numpy as np
        u = np.ascontiguousarray(u, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        if u.size != self.rows * self.cols or v.size != self.rows * self.cols:
            raise ValueError("upload size does not match rows*cols")
        check(self._lib.rdcnn_ring_upload(self._h, u.ctypes.data, v.ctypes.data))

    def upload_ptr(self, u_ptr: int, v_ptr: int):
        check(self._lib.rdcnn_ring_upload(self._h, ctypes.c_void_p(u_ptr), ctypes.c_void_p(v_ptr)))

    def download(self, u=None, v=None):
        import numpy as np
        n = self.rows * self.cols
        u = np.empty(n, np.float32) if u is None else u
        v = np.empty(n, np.float32) if v is None else v
        check(self._lib.rdcnn_ring_download(self._h, u.ctypes.data, v.ctypes.data))
        return u, v

    def download_ptr(self, u_ptr: int, v_ptr: int):
        check(self._lib.rdcnn_ring_download(self._h, ctypes.c_void_p(u_ptr), ctypes.c_void_p(v_ptr)))

    def advance(self, steps: int):
        """Advance every slab; returns first_bad[1]: the exact 1-based
        iteration of the first non-finite value anywhere (0 = finite)."""
        import numpy as np
        bad = ctypes.c_long()
        check(self._lib.rdcnn_ring_advance(self._h, int(steps), ctypes.byref(bad)))
        return np.array([bad.value], dtype=np.int64)

    def elapsed_ms(self) -> float:
        ms = ctypes.c_double()
        check(self._lib.rdcnn_ring_elapsed_ms(self._h, ctypes.byref(ms)))
        return ms.value

    def launch_count(self) -> int:
        n = ctypes.c_long()
        check(self._lib.rdcnn_ring_launch_count(self._h, ctypes.byref(n)))
        return n.value

    def trace_block(self, levels: int = 4):
        """One traced block on every slab: an (n, 6) uint64 array of
        {slab, start ns, end ns, smid, wait ns, peer bytes} per warp."""
        import numpy as np
        cap = 1 << 20
        out = np.zeros((cap, 6), np.uint64)
        n = ctypes.c_longlong()
        check(self._lib.rdcnn_ring_trace_block(self._h, int(levels), out.ctypes.data, cap, ctypes.byref(n)))
        return out[: n.value].copy()


def ring_neighbours(rank: int, world: int):
    """(prev, next): the slab above and the slab below on the periodic ring."""
    return (rank - 1) % world, (rank + 1) % world


def exchange_ops(send_first, send_last, recv_top, recv_bottom, rank: int, world: int):
    """The four point-to-point transfers of one halo exchange, in the order
    they must be issued so that sends and receives between one pair of ranks
    match in issue order even when prev == next (world == 2).

    send_first  -> prev's bottom ghosts     recv_top    <- prev's last rows
    send_last   -> next's top ghosts        recv_bottom <- next's first rows
    """
    prev, nxt = ring_neighbours(rank, world)
    return [("send", send_last, nxt), ("send", send_first, prev),
            ("recv", recv_top, prev), ("recv", recv_bottom, nxt)]


def exchange_halos(send_first, send_last, recv_top, recv_bottom, rank: int, world: int,
                   group=None):
    """Post the halo exchange; returns a list of works to wait on (empty for
    world == 1, where the ring closes on itself and the wrap is a local copy)."""
    if world == 1:
        recv_top.copy_(send_last)
        recv_bottom.copy_(send_first)
        return []
    import torch.distributed as dist

    ops = []
    for kind, tensor, peer in exchange_ops(send_first, send_last, recv_top, recv_bottom, rank, world):
        fn = dist.isend if kind == "send" else dist.irecv
        ops.append(dist.P2POp(fn, tensor, peer, group))
    return dist.batch_isend_irecv(ops)


class SlabStepper:
    """One rank's slab of a global_rows x cols torus on its own GPU."""

    def __init__(self, global_rows: int, cols: int, rank: int, world: int, ghost: int = 4,
                 device: int = 0, mode: str = "strict",
                 exchange: Optional[Callable] = None, seg_rows: int = 0, native: Optional[bool] = None,
                 transport: str = "auto", attach: bool = True, exact_blowup: bool = True):
        """``native`` (default: True unless a Python ``exchange`` is given)
        runs the whole block loop in the C-ABI (rdcnn_slab_advance, no host
        work per block); otherwise each block is driven from Python with
        ``exchange`` (the gloo-testable path).

        ``transport`` (native only): ``"p2p"`` fuses the halo exchange into
        the step kernel -- the edge warps pull the rows beyond the slab
        straight from the neighbours' input buffers over peer memory (CUDA
        IPC), after acquiring their ready words, and publish their own with
        release stores; one launch per block, no ghost-row copies; ``"nccl"`` runs boundary kernel ->
        NCCL send/recv on a comm stream || interior kernel; ``"auto"``
        (default) is p2p unless some rank cannot map its neighbours' memory,
        then NCCL on every rank (``self.transport`` says which).  ``attach=False``
        leaves the ring to the caller (in-process rings, see ``attach_peers``).
        ``exact_blowup`` keeps a recent checkpoint of the slab (teed by the
        first block's kernel, refreshed every 2048 iterations) so a blow-up
        is replayed to its exact iteration (see ``advance``)."""
        if global_rows % world:
            raise ValueError(f"global rows {global_rows} not divisible by world size {world}")
        self._lib = load()
        self.global_rows, self.cols, self.rank, self.world = global_rows, cols, rank, world
        self.rows = global_rows // world
        self.ghost = ghost
        self.device = device
        self.native = (exchange is None) if native is None else native
        self.exchange = exchange or exchange_halos
        self._mode, self._seg_rows = (RDCNN_FAST if mode == "fast" else RDCNN_STRICT), seg_rows
        self.launches = 0
        self._dist_ring = False
        self.exact_blowup = bool(exact_blowup) and self.native
        self._create()
        if transport not in ("p2p", "nccl", "auto"):
            raise ValueError(f"unknown transport {transport!r}")
        self.transport = transport if self.native else "python"
        if self.native and attach:
            if transport == "nccl":
                self._attach_ring()
            elif transport == "p2p":
                self._attach_peers()
            else:
                # auto: the fused peer ring when every rank can map its
                # neighbours' memory, else (on every rank) the NCCL ring.
                if not self._all_ranks(self._try_attach_peers()):
                    self.close()
                    self._create()
                    self._dist_ring = False
                    self._attach_ring()
                    self.transport = "nccl"
                else:
                    self.transport = "p2p"

    def _create(self):
        h = ctypes.c_void_p()
        check(self._lib.rdcnn_slab_create(self.rows, self.cols, self.ghost, self.device, self._mode,
                                          ctypes.byref(h)))
        self._h = h
        check(self._lib.rdcnn_sim_set_tuning(self._h, self.ghost, self._seg_rows))
        if self.exact_blowup:
            check(self._lib.rdcnn_slab_checkpoint_enable(self._h, 1))

    def _all_ranks(self, ok: bool) -> bool:
        if self.world == 1:
            return ok
        import torch
        import torch.distributed as dist

        dev = f"cuda:{self.device}" if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item())

    # -- fused peer ring -------------------------------------------------------
    def export_peer(self) -> "_lib.PeerDesc":
        d = _lib.PeerDesc()
        check(self._lib.rdcnn_slab_peer_export(self._h, ctypes.byref(d)))
        return d

    def attach_peers(self, prev: "_lib.PeerDesc", nxt: "_lib.PeerDesc"):
        check(self._lib.rdcnn_slab_attach_peers(self._h, self.rank, self.world, ctypes.byref(prev),
                                                ctypes.byref(nxt)))

    def _attach_peers(self):
        """Share every rank's peer descriptor (torch.distributed) and open
        the ring neighbours' memory; world 1 closes the ring on itself."""
        mine = self.export_peer()
        if self.world == 1:
            self.attach_peers(mine, mine)
            return
        import torch.distributed as dist

        blobs = [None] * self.world
        dist.all_gather_object(blobs, bytes(mine))
        self._dist_ring = True
        prev, nxt = ring_neighbours(self.rank, self.world)
        self.attach_peers(_lib.PeerDesc.from_buffer_copy(blobs[prev]),
                          _lib.PeerDesc.from_buffer_copy(blobs[nxt]))

    def _try_attach_peers(self) -> bool:
        """_attach_peers that never skips a collective: a rank that cannot
        export or map still joins the descriptor exchange, and reports."""
        try:
            mine = bytes(self.export_peer())
        except Exception:  # noqa: BLE001 - reported through the return value
            mine = None
        if self.world == 1:
            blobs = [mine]
        else:
            import torch.distributed as dist

            blobs = [None] * self.world
            dist.all_gather_object(blobs, mine)
            self._dist_ring = True
        if any(b is None for b in blobs):
            return False
        prev, nxt = ring_neighbours(self.rank, self.world)
        try:
            self.attach_peers(_lib.PeerDesc.from_buffer_copy(blobs[prev]),
                              _lib.PeerDesc.from_buffer_copy(blobs[nxt]))
        except Exception:  # noqa: BLE001 - reported through the return value
            return False
        return True

    def _attach_ring(self):
        """NCCL communicator for the ring (id from rank 0, shared through
        torch.distributed); world 1 needs none."""
        uid = (ctypes.c_uint8 * 128)()
        if self.world > 1:
            import torch
            import torch.distributed as dist
            if self.rank == 0:
                check(self._lib.rdcnn_nccl_unique_id(uid))
            on_gpu = dist.get_backend() == "nccl"
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8,
                             device=f"cuda:{self.device}" if on_gpu else "cpu")
            dist.broadcast(t, src=0)
            for k, b in enumerate(t.cpu().tolist()):
                uid[k] = b
        check(self._lib.rdcnn_slab_attach_ring(self._h, uid, self.rank, self.world))

    def elapsed_ms(self) -> float:
        ms = ctypes.c_double()
        check(self._lib.rdcnn_sim_elapsed_ms(self._h, ctypes.byref(ms)))
        return ms.value

    def close(self):
        if getattr(self, "_h", None):
            self._lib.rdcnn_sim_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- state ---------------------------------------------------------------
    def init(self, typ: int, seed: int):
        check(self._lib.rdcnn_slab_init(self._h, typ, ctypes.c_uint64(seed), self.global_rows,
                                        self.rank * self.rows))

    def set_params(self, gene):
        from .engine import params_from_gene
        p = params_from_gene(gene)
        check(self._lib.rdcnn_sim_set_params(self._h, ctypes.byref(p), 1))

    def upload(self, u, v):
        import numpy as np
        u = np.ascontiguousarray(u, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        check(self._lib.rdcnn_sim_upload(self._h, u.ctypes.data, v.ctypes.data))

    def download(self):
        import numpy as np
        n = self.rows * self.cols
        u = np.empty(n, np.float32)
        v = np.empty(n, np.float32)
        check(self._lib.rdcnn_sim_download(self._h, u.ctypes.data, v.ctypes.data))
        return u, v

    def _views(self, which: int):
        import torch

        first, ghost0 = ctypes.c_void_p(), ctypes.c_void_p()
        check(self._lib.rdcnn_slab_rows_ptr(self._h, which, ctypes.byref(first), ctypes.byref(ghost0)))
        g, w = self.ghost, 2 * self.cols
        bpr = 4 * w  # bytes per interleaved row
        dev = f"cuda:{self.device}"
        as_t = lambda ptr: torch.as_tensor(_CudaRows(ptr, g, w), device=dev)  # noqa: E731
        send_first = as_t(first.value)
        send_last = as_t(first.value + (self.rows - g) * bpr)
        recv_top = as_t(ghost0.value)
        recv_bottom = as_t(first.value + self.rows * bpr)
        return send_first, send_last, recv_top, recv_bottom

    # -- stepping ------------------------------------------------------------
    def fill_ghosts(self):
        """Exchange the front buffer's edge rows (before the first block)."""
        import torch

        if self.native:
            p2p_ring = self._dist_ring  # ranks in separate processes
            if p2p_ring:
                import torch.distributed as dist
                dist.barrier()  # no rank still reads the ghosts this overwrites
            check(self._lib.rdcnn_slab_fill_ghosts(self._h))
            if p2p_ring:
                dist.barrier()  # every ghost row is in before any rank's first block
            return
        works = self.exchange(*self._views(0), self.rank, self.world)
        for w in works:
            w.wait()
        torch.cuda.current_stream(self.device).synchronize()

    # -- blow-up (engine.hpp:79, BlowUpError(iter + 1)) -----------------------
    def _advance_native(self, steps: int) -> int:
        """One native advance; the first iteration (1-based) of this rank's
        first bad block, or 0."""
        bad = ctypes.c_long()
        rc = self._lib.rdcnn_slab_advance(self._h, int(steps), ctypes.byref(bad))
        if rc != _lib.RDCNN_EBLOWUP:
            check(rc)
        n = ctypes.c_long()
        check(self._lib.rdcnn_sim_launch_count(self._h, ctypes.byref(n)))
        self.launches += n.value
        return bad.value if rc == _lib.RDCNN_EBLOWUP else 0

    def _agree(self, x: int, op: str) -> int:
        """min over ranks of the non-zero values (0 = none), or max."""
        if not self._dist_ring:
            return x
        import torch
        import torch.distributed as dist

        big = 1 << 62
        dev = f"cuda:{self.device}" if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([(x or big) if op == "min" else x], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN if op == "min" else dist.ReduceOp.MAX)
        v = int(t.item())
        return 0 if (op == "min" and v == big) else v

    def _replay_exact(self, first_block_iter: int) -> int:
        """Every rank: restore the checkpoint (``age`` iterations before this
        advance's input; the same on every rank), re-run to the first bad
        block, then one level at a time until any rank flags.  Leaves the
        post-blow-up state (as run_timed does, engine.hpp:103-104) and returns
        the exact 1-based iteration within this advance."""
        age = ctypes.c_long()
        check(self._lib.rdcnn_slab_checkpoint_age(self._h, ctypes.byref(age)))
        check(self._lib.rdcnn_slab_restore(self._h))
        # Every rank has restored before any rank's replay reads its
        # neighbours' rows: their ready words still carry the last block of
        # the advance, so without this a fast rank could pull a neighbour's
        # post-blow-up rows (seen as a rare 3-process IPC failure).
        self._agree(0, "max")
        pre = age.value + first_block_iter - 1
        if pre and self._agree(self._advance_native(pre), "min"):
            raise RuntimeError("blow-up before the first flagged block on replay")
        for m in range(1, self.ghost + 1):
            if self._agree(1 if self._advance_native(1) else 0, "max"):
                return first_block_iter - 1 + m
        raise RuntimeError(f"blow-up flagged in the block at iteration {first_block_iter} "
                           "was not reproduced by the replay")

    def advance(self, steps: int, stream=None):
        """Advance by `steps` iterations in blocks of <= ghost levels.

        Native path: returns 0, or the exact first iteration (1-based, as
        BlowUpError.iteration) at which any rank's slab held a non-finite
        value -- agreed over the ranks, found by replaying the first bad block
        level by level from the advance's checkpointed input (block
        granularity with ``exact_blowup=False``)."""
        import torch

        if self.native:
            first = self._agree(self._advance_native(steps), "min")
            if first == 0 or not self.exact_blowup:
                return first
            return self._replay_exact(first)
        st = stream or torch.cuda.current_stream(self.device)
        sp = ctypes.c_void_p(st.cuda_stream)
        done = 0
        while done < steps:
            k = self.ghost
            while k > steps - done:
                k //= 2
            check(self._lib.rdcnn_slab_step_boundary(self._h, k, sp))
            works = self.exchange(*self._views(1), self.rank, self.world)
            check(self._lib.rdcnn_slab_step_interior(self._h, k, sp))
            for w in works:
                w.wait()
            check(self._lib.rdcnn_slab_swap(self._h))
            self.launches += 3
            done += k

    def blew_up(self) -> bool:
        bad = ctypes.c_int()
        check(self._lib.rdcnn_slab_poll_blowup(self._h, ctypes.byref(bad), None))
        return bool(bad.value)
