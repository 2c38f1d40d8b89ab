"""The Schwarz coupler's distributed receiver logic (R21) on the CPU, world size 2 over gloo:
each rank runs the library's own host routine (osmpm_schwarz_receivers_host, the code the coupler calls
per slab) on its slab of the fine node box -- owned planes plus the two ghost planes its stencils
reach -- the coarse nodes taken over by fine donors are OR-ed over the ranks (the NCCL max of the GPU
path, here gloo), and the result must equal the undecomposed decision and the oracle's receivers
(oracle.schwarz.receivers, an independent Python implementation of PAPER.md:283-303)."""
import ctypes as C
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_2605_09097_b200 import build
    lib = C.CDLL(build.build())
    lib.osmpm_last_error.restype = C.c_char_p
    return lib


def _desc(grid):
    from paper_2605_09097_b200.osmpm import grid_desc
    return grid_desc(grid)


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def box_receivers(coarse_grid, mB, gB, aB, fine_grid, lo, dims, nown, mS, mbS, aS, tauS, drop):
    """One call of the library routine over a fine box [lo, lo + dims) (arrays over that box)."""
    lib = _lib()
    cd, fd = _desc(coarse_grid), _desc(fine_grid)
    clo = (C.c_int64 * 3)(0, 0, 0)
    cdims = (C.c_int64 * 3)(*[coarse_grid.dims[a] for a in range(3)])
    flo = (C.c_int64 * 3)(*lo)
    fdims = (C.c_int64 * 3)(*dims)
    cap = int(np.prod([d for d in dims if d > 0]))
    recv = np.zeros(cap, np.int64)
    own = np.zeros(cap, np.uint8)
    n = C.c_int64()
    rc = lib.osmpm_schwarz_receivers_host(
        C.byref(cd), clo, cdims, _p(mB), _p(gB), _p(aB), C.byref(fd), flo, fdims, C.c_int64(nown), _p(mS), _p(mbS),
        _p(aS), C.c_double(tauS), _p(drop), C.c_int64(cap), _p(recv), _p(own), C.byref(n))
    assert rc == 0, lib.osmpm_last_error()
    return recv[: n.value], own[: n.value].astype(bool)


def _inputs():
    """C1 (BASELINE configs[0]) at rest: the arrays the coupler reads back after its step-0 P2G."""
    import oracle
    import synth
    coarse, fine = synth.c1_cantilever()
    gsB, gsS = oracle.p2g(coarse), oracle.p2g(fine)
    tauB = 1e-6 * oracle.median(coarse.particles.m)
    tauS = 1e-6 * oracle.median(fine.particles.m)
    mbB, mbS = oracle.boundary_mass(coarse), oracle.boundary_mass(fine)
    gB = (gsB.active.astype(bool) & (mbB > tauB)).astype(np.uint8)
    return coarse, fine, gsB, gsS, gB, mbS, tauB, tauS


def _slab(fine, arrs, x0, x1, ghost):
    """arrays of the fine box restricted to node planes [x0, x1) (+ ghost planes), C order, x slowest"""
    nx, ny = fine.grid.dims[0], fine.grid.dims[1]
    hi = min(x1 + ghost, nx)
    out = [np.ascontiguousarray(a.reshape(nx, ny)[x0:hi].reshape(-1)) for a in arrs]
    return out, (x0, 0, 0), (hi - x0, ny, 1), (x1 - x0) * ny


def test_undecomposed_matches_the_oracle():
    from oracle import schwarz as OS
    import oracle
    coarse, fine, gsB, gsS, gB, mbS, tauB, tauS = _inputs()
    drop = np.zeros_like(gB)
    nx, ny = fine.grid.dims[0], fine.grid.dims[1]
    recv, own = box_receivers(coarse.grid, gsB.m, gB, gsB.active, fine.grid, (0, 0, 0), (nx, ny, 1), nx * ny,
                              gsS.m, mbS, gsS.active, tauS, drop)
    hatB, hatS = OS.receivers(coarse, fine, gsB, gsS, 1e-6)
    assert own.all()
    np.testing.assert_array_equal(recv, np.flatnonzero(hatS))
    _, _, den = oracle.project(fine.grid, gsS, coarse.grid, 0.0)
    np.testing.assert_array_equal(gB.astype(bool) & ~drop.astype(bool) & (den > tauB), hatB)
    assert drop.sum() > 0 and recv.size > 0  # the C1 overlap has ambiguous nodes and receivers


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cut, q):
    try:
        import torch
        import torch.distributed as dist
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        coarse, fine, gsB, gsS, gB, mbS, tauB, tauS = _inputs()
        nx = fine.grid.dims[0]
        x0, x1 = (0, cut) if rank == 0 else (cut, nx)
        (mS, mb, aS), lo, dims, nown = _slab(fine, (gsS.m, mbS, gsS.active), x0, x1, 2 if rank == 0 else 0)
        drop = np.zeros_like(gB)
        recv, own = box_receivers(coarse.grid, gsB.m, gB, gsB.active, fine.grid, lo, dims, nown, mS, mb, aS, tauS,
                                  drop)
        t = torch.from_numpy(drop.astype(np.int32))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # the NCCL max over ranks of the GPU path
        q.put((rank, recv.tolist(), own.tolist(), t.numpy().astype(np.uint8).tolist()))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, "error", repr(e), None))


def test_two_rank_receivers_equal_the_undecomposed_decision():
    import torch.multiprocessing as mp
    coarse, fine, gsB, gsS, gB, mbS, tauB, tauS = _inputs()
    nx, ny = fine.grid.dims[0], fine.grid.dims[1]
    drop_ref = np.zeros_like(gB)
    recv_ref, _ = box_receivers(coarse.grid, gsB.m, gB, gsB.active, fine.grid, (0, 0, 0), (nx, ny, 1), nx * ny,
                                gsS.m, mbS, gsS.active, tauS, drop_ref)
    # cut the x node planes one plane into the receiver band, so that rank 0's ghost planes hold receivers
    cut = int((recv_ref // ny).min()) + 1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cut, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        item = q.get(timeout=300)
        assert item[1] != "error", item
        res[item[0]] = item
    for p in procs:
        p.join(timeout=60)
    owned = [set(np.asarray(res[r][1])[np.asarray(res[r][2], bool)]) for r in range(2)]
    ghosts0 = set(np.asarray(res[0][1])[~np.asarray(res[0][2], bool)])
    assert owned[0].isdisjoint(owned[1])
    assert owned[0] | owned[1] == set(recv_ref.tolist())
    # rank 0's ghost planes carry exactly rank 1's decisions for those nodes
    ghost_nodes = {g for g in owned[1] if g // ny < cut + 2}
    assert ghosts0 == ghost_nodes and len(ghosts0) > 0
    # the OR over ranks of the coarse take-overs equals the undecomposed one, on both ranks
    for r in range(2):
        np.testing.assert_array_equal(np.asarray(res[r][3], np.uint8), drop_ref)
