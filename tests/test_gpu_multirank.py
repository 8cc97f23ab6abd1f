"""Destination-range partitioning through the real device engine: two rank
processes share the one B200 of a gpurun box and exchange layer outputs
(and transform-first z rows, and GAT z rows) with gloo collectives on CUDA
tensors -- the same Engine code the 8-GPU NCCL job runs (runtime.py
gather_ranges / allreduce_max). The reassembled output must equal the
single-rank engine's bit for bit: every layer's rows depend only on the
rows gathered before it, and both paths run the same kernels per row."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = Path(__file__).resolve().parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case(model):
    from paper_2605_09402_b200 import storage as S
    graph, feats = S.synthetic_in_memory("uniform", 6007, 7, 64, 13)
    if model == "gat":
        from paper_2605_09402_b200.gat import random_gat_weights
        return graph, feats.astype(np.float16), \
            random_gat_weights([64, 32, 5], 4, seed=5)
    kind = {"gcn": 0, "sage": 1, "gin": 2}[model]
    # [64, 48, 12]: layer 1 aggregate-first, layer 2 transform-first
    return graph, feats, S.random_weights(S.ModelKind(kind), [64, 48, 12], 5,
                                          gin_epsilon=0.25)


def _engine(model, graph, w, backend, rank, world, group=None):
    from paper_2605_09402_b200.runtime import Engine, PipelineConfig
    cfg = PipelineConfig(backend=backend, hot_slots=6007,
                         chunk_budget=32 << 10)
    if model == "gat":
        from paper_2605_09402_b200.gat import GATEngine
        return GATEngine(graph, w, cfg, rank=rank, world=world,
                         dist_group=group)
    return Engine(graph, w, cfg, rank=rank, world=world, dist_group=group)


def _worker(rank, world, port, model, backend, q, own=False):
    sys.path.insert(0, str(HERE.parent))
    sys.path.insert(0, str(HERE))
    import torch
    import torch.distributed as dist
    from paper_2605_09402_b200.runtime import gather_ranges
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        graph, feats, w = _case(model)
        eng = _engine(model, graph, w, backend, rank, world,
                      dist.group.WORLD)
        # own=True: the rank holds only its partition of the input, in
        # pinned host memory (the engine uploads and all-gathers it)
        x = torch.as_tensor(feats[eng.lo:eng.hi]).pin_memory() if own \
            else torch.as_tensor(feats).cuda()
        y, metrics = eng.infer(x)
        full = gather_ranges(y, eng.ranges)
        q.put((rank, full.cpu().numpy() if rank == 0 else None,
               sum(m.messages for m in metrics)))
        eng.close()
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("model,backend,own", [("gcn", "stable", False),
                                               ("sage", "tcgen05", False),
                                               ("gin", "tcgen05", False),
                                               ("gat", "tcgen05", False),
                                               ("gcn", "tcgen05", True),
                                               ("sage", "tcgen05", True)])
def test_two_ranks_on_one_gpu_match_single_rank(model, backend, own):
    import torch
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker,
                         args=(r, 2, port, model, backend, q, own))
             for r in range(2)]
    for p in procs:
        p.start()
    got = sorted((q.get(timeout=600) for _ in procs), key=lambda g: g[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    graph, feats, w = _case(model)
    eng = _engine(model, graph, w, backend, 0, 1)
    y1, m1 = eng.infer(torch.as_tensor(feats).cuda())
    np.testing.assert_array_equal(got[0][1], y1.cpu().numpy())
    # every in-edge (+ self term) is delivered exactly once over the ranks
    assert got[0][2] + got[1][2] == sum(m.messages for m in m1)
    eng.close()
