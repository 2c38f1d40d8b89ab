"""CPU tests of the host logic of the multi-GPU path, world size 2
over the gloo backend (no GPU):

* the slab cuts (osmpm_slab_cuts, the exact routine the decomposed subdomain uses at creation) are
  tile-aligned, increasing, balanced, and identical on every rank given the same particles, so the
  ranks' particle sets partition the whole set;
* bench.py's process-group plumbing: rank 0's communicator id reaches every rank, timings are the
  max over ranks, only rank 0 prints, the reference arm runs on rank 0 only.
"""
import ctypes
import io
import json
import os
import socket
import sys
from contextlib import redirect_stdout

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_2605_09097_b200 import build
    lib = ctypes.CDLL(build.build())
    lib.osmpm_last_error.restype = ctypes.c_char_p
    return lib


def slab_cuts(base_x, nslab, tile):
    lib = _lib()
    bx = np.ascontiguousarray(base_x, dtype=np.int32)
    cuts = np.zeros(max(nslab - 1, 1), dtype=np.int32)
    rc = lib.osmpm_slab_cuts(bx.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(bx.size), ctypes.c_int32(nslab),
                             ctypes.c_int32(tile), cuts.ctypes.data_as(ctypes.c_void_p))
    if rc != 0:
        raise ValueError(lib.osmpm_last_error().decode())
    return cuts[: nslab - 1]


def owner(base_x, cuts):
    return np.searchsorted(np.asarray(cuts), np.asarray(base_x), side="right")


@pytest.mark.parametrize("nslab,tile", [(2, 4), (3, 4), (8, 4), (4, 16)])
def test_cuts_aligned_increasing_balanced(nslab, tile):
    rng = np.random.default_rng(nslab * 31 + tile)
    # C5-like: a uniform block of cells at 8 particles per cell, offset from 0
    base = np.repeat(np.arange(100, 100 + 64), 8)
    base = np.concatenate([base, rng.integers(100, 164, size=333)])
    cuts = slab_cuts(base, nslab, tile)
    assert len(cuts) == nslab - 1
    assert np.all(np.diff(cuts) > 0)
    assert np.all((cuts - base.min()) % tile == 0)
    counts = np.bincount(owner(base, cuts), minlength=nslab)
    assert counts.sum() == base.size and np.all(counts > 0)
    # balanced to within one tile column of particles
    col = np.bincount((base - base.min()) // tile).max()
    assert np.abs(counts - base.size / nslab).max() <= col


def test_cuts_skewed_density_and_errors():
    # a dense cluster on the left: cuts move left to balance the counts
    base = np.concatenate([np.repeat(np.arange(0, 16), 40), np.repeat(np.arange(16, 64), 2)])
    cuts = slab_cuts(base, 2, 4)
    counts = np.bincount(owner(base, cuts), minlength=2)
    assert cuts[0] < 32 and abs(counts[0] - counts[1]) <= 4 * 40
    with pytest.raises(ValueError):
        slab_cuts(np.arange(0, 8), 3, 4)  # 2 tile columns, 3 slabs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        sys.path.insert(0, ROOT)
        import bench
        # the decomposition's cuts agree on every rank; ownership partitions the particles
        rng = np.random.default_rng(7)  # identical particle view on every rank
        base = rng.integers(40, 200, size=5000)
        cuts = slab_cuts(base, 2 * world, 4)
        allc = [None] * world
        dist.all_gather_object(allc, cuts.tolist())
        own = owner(base, cuts)
        mine = np.isin(own, [2 * rank, 2 * rank + 1]).sum()
        tot = bench.sum_over_ranks(dist, mine, "cpu")
        # communicator id from rank 0
        uid = bench.share_unique_id(dist, rank, lambda: bytes(range(128)))
        # max over ranks of a per-rank timing
        tmax = bench.max_over_ranks(dist, 10.0 + rank, "cpu")
        # reference arm: rank 0 alone prints one line
        args = type("A", (), dict(cpu_cells=3, warmup=0, steps=1, newton=1, cg=2, gpus=world))()
        buf = io.StringIO()
        with redirect_stdout(buf):
            bench.run_reference(args, rank)
        q.put((rank, allc, tot, uid, tmax, buf.getvalue()))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, "error", repr(e)))


def test_two_rank_gloo_plumbing():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        item = q.get(timeout=300)
        assert item[1] != "error", item
        res[item[0]] = item
    for p in procs:
        p.join(timeout=60)
    (_, c0, t0, u0, m0, o0), (_, c1, t1, u1, m1, o1) = res[0], res[1]
    assert c0 == c1 and c0[0] == c0[1]
    assert t0 == t1 == 5000
    assert u0 == u1 == bytes(range(128))
    assert m0 == m1 == 11.0
    assert o1 == ""
    line = json.loads(o0)
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "oracle"
