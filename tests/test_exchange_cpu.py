"""The multi-GPU exchange (paper_2605_09402_b200/exchange.py)
on CPU: the piece schedule, and gloo process groups of 2 and 3 ranks whose
owner broadcasts fill one (V, width) buffer in place. The same code runs
NCCL over NVLink on a multi-GPU box."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2605_09402_b200.exchange import RangeExchange
from paper_2605_09402_b200.storage import partition_ranges

HERE = Path(__file__).resolve().parent


@pytest.mark.parametrize("v,g,pieces", [(10, 3, 4), (2, 3, 2), (1000, 8, 4),
                                        (7, 1, 3), (0, 2, 2)])
def test_schedule_tiles_rows_in_ascending_order(v, g, pieces):
    ranges = partition_ranges(v, g)
    for rank in range(g):
        ex = RangeExchange(v, ranges, rank, pieces_per_rank=pieces,
                           min_piece_bytes=1)
        sched = ex.schedule(row_bytes=16)
        rows = [r for _, a, b in sched for r in range(a, b)]
        assert rows == list(range(v))
        for owner, a, b in sched:
            lo, hi = ranges[owner]
            assert lo <= a < b <= hi
        per_owner = {}
        for owner, _, _ in sched:
            per_owner[owner] = per_owner.get(owner, 0) + 1
        assert all(n <= pieces for n in per_owner.values())


def test_schedule_respects_min_piece_bytes():
    ranges = partition_ranges(1000, 2)
    ex = RangeExchange(1000, ranges, 0, pieces_per_rank=8,
                       min_piece_bytes=100 * 64)
    sched = ex.schedule(row_bytes=64)
    assert len(sched) == 2 * 5  # 500 rows x 64 B per owner / 6400 B


def _worker(rank, world, port, v, width, q):
    sys.path.insert(0, str(HERE.parent))
    import torch
    import torch.distributed as dist
    from paper_2605_09402_b200.exchange import RangeExchange, gather_ranges
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ranges = partition_ranges(v, world)
        ex = RangeExchange(v, ranges, rank, None, pieces_per_rank=3,
                           min_piece_bytes=1)
        full = ex.buffer("h", width, torch.float32, "cpu")
        full.fill_(-1.0)
        lo, hi = ranges[rank]
        own = ex.own(full)
        own.copy_(torch.arange(lo * width, hi * width,
                               dtype=torch.float32).reshape(-1, width))
        bounds, events = ex.start(full)
        ex.finish(events)
        # the same buffer object is filled (no copy, no concatenation)
        assert ex.buffer("h", width, torch.float32, "cpu") is full
        local = torch.full((hi - lo, 2), float(rank))
        g = gather_ranges(local, ranges)
        q.put((rank, full.numpy().copy(), bounds.tolist(),
               ex.bytes_received, g.numpy().copy()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,v", [(2, 1201), (3, 10), (3, 2)])
def test_gloo_owner_broadcasts_fill_buffer_in_place(world, v):
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    width = 5
    procs = [ctx.Process(target=_worker, args=(r, world, port, v, width, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = sorted((q.get(timeout=300) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.arange(v * width, dtype=np.float32).reshape(v, width)
    ranges = partition_ranges(v, world)
    owner_of = np.concatenate([np.full(hi - lo, g, np.float32)
                               for g, (lo, hi) in enumerate(ranges)])
    for rank, full, bounds, received, gathered in got:
        np.testing.assert_array_equal(full, want)
        assert bounds[0] == 0 and bounds[-1] == v
        assert bounds == sorted(bounds)
        lo, hi = ranges[rank]
        assert received == (v - (hi - lo)) * width * 4
        np.testing.assert_array_equal(gathered[:, 0], owner_of)
