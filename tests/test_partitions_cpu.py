"""Destination-range partitioning on CPU.

* the per-range integer machine of the oracle is pinned against a harness
  that drives the reference's own MemoryManager + policies (unchanged,
  imported) with the A.1 procedure restricted to [lo, hi);
* a world_size-2 gloo job runs one range per rank and reassembles the
  next layer's input with ``runtime.gather_ranges`` (the NCCL all-gather
  of the GPU path); the result equals the single-process layer bit-exactly.
"""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

from helpers import REFERENCE_SRC
from paper_2605_09402_b200 import storage as S
from paper_2605_09402_b200.storage import partition_ranges


def oracle_range(graph, feats, w, l, rows, slots, rng_range, eviction="minpend"):
    from oracle import engine as OE
    lw = w.layers[l]
    return OE.run_layer(graph.offsets, graph.neighbors, graph.in_degrees,
                        feats, int(w.kind), lw.weight, lw.bias, relu=True,
                        embed_dim=w.embedding_dim(l), agg_dim=w.agg_dim(l),
                        chunk_rows=rows, slot_count=slots,
                        gin_epsilon=w.gin_epsilon, eviction=eviction,
                        dst_range=rng_range)


def reference_range_harness(graph, feats, w, rows, slots, lo, hi):
    """A.1 restricted to [lo, hi), driving oocgnn's MemoryManager."""
    sys.path.insert(0, str(REFERENCE_SRC))
    from oocgnn.iostats import IOCounters, StageCounters
    from oocgnn.memstore import MemoryBudget, MemoryManager, make_policy
    from oocgnn.vertexstate import NOT_STARTED, StateTable
    import tempfile

    kind = int(w.kind)
    v = graph.num_vertices
    indeg = graph.in_degrees
    pending = indeg.astype(np.uint32) + np.uint32(kind != 0)
    states = StateTable(v)
    victims, grads = [], []
    pol = make_policy("minpend", int(pending.max()), 0)
    choose = pol.choose_victims

    def rec(k):
        got = choose(k)
        victims.append(list(got))
        return got
    pol.choose_victims = rec
    cold = Path(tempfile.mkdtemp()) / "cold.bin"
    mem = MemoryManager(MemoryBudget(slots, w.agg_dim(0)), pending, states,
                        pol, cold, IOCounters(), StageCounters())
    sub = max(1, slots // 2)

    def deliver(vs, cnt):
        for a in range(0, len(vs), sub):
            b_ = vs[a:a + sub]
            c_ = cnt[a:a + sub]
            mem.ensure_hot_many(b_)
            pending[b_] -= c_.astype(np.uint32)
            for x, p in zip(b_.tolist(), pending[b_].tolist()):
                pol.on_message(x, int(p))
            done = b_[pending[b_] == 0]
            if done.size:
                mem.release_batch(done)
                grads.append(done.tolist())

    for s in range(0, v, rows):
        e = min(s + rows, v)
        src = np.arange(s, e)
        mine = src[(src >= lo) & (src < hi)]
        if kind == 1:  # SAGE self pass
            deliver(mine, np.ones(len(mine), np.int64))
        elif kind == 0:
            zeros = mine[(states.array[mine] == NOT_STARTED)
                         & (pending[mine] == 0)]
            for a in range(0, len(zeros), sub):
                z = zeros[a:a + sub]
                mem.ensure_hot_many(z)
                mem.release_batch(z)
                grads.append(z.tolist())
        o0, o1 = int(graph.offsets[s]), int(graph.offsets[e])
        fan = np.diff(graph.offsets[s:e + 1])
        if kind == 2:  # GIN: self term before each source's edges
            dst = np.concatenate([np.concatenate(([u], graph.neighbors[
                graph.offsets[u]:graph.offsets[u + 1]])) for u in src]) \
                if len(src) else np.empty(0, np.int64)
        else:
            dst = graph.neighbors[o0:o1]
        order = np.argsort(dst, kind="stable")
        uniq, seg = np.unique(dst[order], return_index=True)
        cnt = np.diff(np.append(seg, len(dst)))
        first = order[seg]
        keep = (uniq >= lo) & (uniq < hi)
        app = np.argsort(first[keep], kind="stable")
        deliver(uniq[keep][app], cnt[keep][app])
    mem.close()
    return victims, grads, mem.counters


@pytest.mark.skipif(not REFERENCE_SRC.exists(), reason="reference absent")
@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("parts", [2, 3])
def test_range_oracle_pinned_to_reference_memory_manager(kind, parts):
    graph, feats = S.synthetic_in_memory("uniform", 1500, 6, 8, 3)
    w = S.random_weights(S.ModelKind(kind), [8, 4], 5, gin_epsilon=0.1)
    rows, slots = 97, 24
    for lo, hi in partition_ranges(graph.num_vertices, parts):
        _, m, log = oracle_range(graph, feats, w, 0, rows, slots, (lo, hi))
        victims, grads, counters = reference_range_harness(
            graph, feats, w, rows, slots, lo, hi)
        assert log.victims == victims
        assert log.graduated == grads
        assert m.evictions == counters.evictions
        assert m.reloads == counters.reloads
        assert m.hot_peak == counters.hot_peak


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from paper_2605_09402_b200.runtime import gather_ranges
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    graph, feats = S.synthetic_in_memory("uniform", 1201, 5, 8, 4)
    w = S.random_weights(S.ModelKind.SAGE, [8, 4], 5)
    ranges = partition_ranges(graph.num_vertices, world)
    y, m, _ = oracle_range(graph, feats, w, 0, 200, 10_000, ranges[rank])
    full = gather_ranges(torch.from_numpy(y), ranges)
    if rank == 0:
        q.put((full.numpy(), m.messages))
    else:
        q.put((None, m.messages))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_reassemble_layer():
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q))
             for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = next(g[0] for g in got if g[0] is not None)
    graph, feats = S.synthetic_in_memory("uniform", 1201, 5, 8, 4)
    w = S.random_weights(S.ModelKind.SAGE, [8, 4], 5)
    y1, m1, _ = oracle_range(graph, feats, w, 0, 200, 10_000, None)
    np.testing.assert_array_equal(full, y1)
    # every in-range edge + self term is delivered exactly once overall
    assert sum(g[1] for g in got) == m1.messages
