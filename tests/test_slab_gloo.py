"""Multi-process (world_size 2 and 3, gloo on CPU) test of the row-slab ring
halo exchange that the multi-GPU path runs over NCCL (slab.py).

Each rank owns rows [r*S, (r+1)*S) of a global torus; after one exchange its
top ghosts must hold the previous rank's last rows and its bottom ghosts the
next rank's first rows (the torus row wrap of reference kernels.hpp:46-47).
A second test steps a whole torus with slabs + exchanges, using the CPU
oracle as the per-slab stepper, and checks the result equals the unsplit
torus bit for bit -- the same decomposition the GPU path uses.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2102_10340_b200.slab import exchange_halos, exchange_ops, ring_neighbours


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _exchange_worker(rank, world, port, ghost, cols, errq):
    try:
        _init(rank, world, port)
        S = 5
        # Interleaved slab rows (u then v per row) with ghosts, as on the GPU.
        buf = torch.full((S + 2 * ghost, 2 * cols), -1.0)
        for i in range(S):
            buf[ghost + i] = float(rank * S + i)
        views = (buf[ghost:2 * ghost], buf[S:S + ghost], buf[0:ghost], buf[S + ghost:S + 2 * ghost])
        send_first, send_last, recv_top, recv_bottom = [v.clone() for v in views]
        works = exchange_halos(send_first, send_last, recv_top, recv_bottom, rank, world)
        for w in works:
            w.wait()
        rows_global = world * S
        for g in range(ghost):
            want_top = (rank * S - ghost + g) % rows_global
            want_bot = (rank * S + S + g) % rows_global
            assert torch.all(recv_top[g] == want_top), (rank, g, recv_top[g][0].item(), want_top)
            assert torch.all(recv_bottom[g] == want_bot), (rank, g, recv_bottom[g][0].item(), want_bot)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        errq.put(f"rank {rank}: {e!r}")
        raise


def _torus_worker(rank, world, port, ghost, rows, cols, iters, errq):
    try:
        from oracle.oracle import Oracle
        _init(rank, world, port)
        orc = Oracle()
        u0, v0 = orc.init(2, rows, cols, 9)
        S = rows // world
        U = u0.reshape(rows, cols)[rank * S:(rank + 1) * S].copy()
        V = v0.reshape(rows, cols)[rank * S:(rank + 1) * S].copy()
        done = 0
        while done < iters:
            k = min(ghost, iters - done)
            # ghost exchange of depth k (rows packed u|v per row like the GPU layout)
            own = np.concatenate([U, V], axis=1)
            send_first = torch.from_numpy(own[:k].copy())
            send_last = torch.from_numpy(own[S - k:].copy())
            recv_top = torch.empty_like(send_first)
            recv_bottom = torch.empty_like(send_last)
            for w in exchange_halos(send_first, send_last, recv_top, recv_bottom, rank, world):
                w.wait()
            ext = np.concatenate([recv_top.numpy(), own, recv_bottom.numpy()], axis=0)
            EU, EV = ext[:, :cols], ext[:, cols:]
            # k steps on the extended slab; rows within k of the (non-periodic)
            # edge are garbage after k steps, the owned rows are exact.
            # The oracle is periodic, so embed the slab in a taller torus
            # padded far enough that the wrap never reaches the owned rows.
            pad = k + 1
            H = S + 2 * k + 2 * pad
            PU = np.zeros((H, cols), np.float32)
            PV = np.zeros((H, cols), np.float32)
            PU[pad:pad + S + 2 * k] = EU
            PV[pad:pad + S + 2 * k] = EV
            ru, rv, bad = orc.run(H, cols, PU, PV, k)
            assert bad == 0
            U = ru.reshape(H, cols)[pad + k:pad + k + S].copy()
            V = rv.reshape(H, cols)[pad + k:pad + k + S].copy()
            done += k
        gu = [torch.zeros(S, cols) for _ in range(world)]
        gv = [torch.zeros(S, cols) for _ in range(world)]
        dist.all_gather(gu, torch.from_numpy(U))
        dist.all_gather(gv, torch.from_numpy(V))
        if rank == 0:
            want_u, want_v, _ = orc.run(rows, cols, u0, v0, iters)
            got_u = torch.cat(gu).numpy().reshape(-1)
            got_v = torch.cat(gv).numpy().reshape(-1)
            assert np.array_equal(got_u.view(np.uint32), want_u.view(np.uint32))
            assert np.array_equal(got_v.view(np.uint32), want_v.view(np.uint32))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        errq.put(f"rank {rank}: {e!r}")
        raise


def _spawn(fn, world, *args):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, *args, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errors = []
    while not errq.empty():
        errors.append(errq.get())
    assert not errors, errors
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


def test_ring_neighbours_and_order():
    assert ring_neighbours(0, 4) == (3, 1)
    assert ring_neighbours(3, 4) == (2, 0)
    ops = exchange_ops("F", "L", "T", "B", 0, 2)
    # with world=2 prev == next: sends (last, first) and receives (top, bottom)
    # must pair in issue order: last -> peer's top, first -> peer's bottom
    assert [o[:2] for o in ops] == [("send", "L"), ("send", "F"), ("recv", "T"), ("recv", "B")]


def test_world1_exchange_is_local_wrap():
    S, g, c = 6, 2, 3
    own = torch.arange(S * c, dtype=torch.float32).reshape(S, c)
    top, bot = torch.empty(g, c), torch.empty(g, c)
    assert exchange_halos(own[:g], own[S - g:], top, bot, 0, 1) == []
    assert torch.equal(top, own[S - g:]) and torch.equal(bot, own[:g])


@pytest.mark.parametrize("world,ghost", [(2, 1), (2, 4), (3, 2)])
def test_gloo_halo_exchange(world, ghost):
    _spawn(_exchange_worker, world, ghost, 7)


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_slab_decomposition_matches_torus(world):
    _spawn(_torus_worker, world, 4, 12 * world, 20, 11)
