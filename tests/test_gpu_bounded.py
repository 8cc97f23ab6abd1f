"""Bounded device records (PipelineConfig.bound_records,
atlas_layer_run_blocked): destinations aggregate and transform in blocks of
the slot budget, so at most slot_count x agg_dim f32 records are ever
resident -- the reference's graduated batches leaving the hot store
(oocgnn/compute.py:125-205, oocgnn/memstore.py:479-494). Every golden case
must stay bit-exact (stable backend) with the reference's integers,
including the cold-store byte counters, and the records must fit the
budget."""

import numpy as np
import pytest
import torch

from helpers import case_config, case_weights, dataset, digest_array, \
    golden_manifest
from paper_2605_09402_b200.runtime import Engine, PipelineConfig

pytestmark = pytest.mark.gpu

CASES = sorted(k for k in golden_manifest() if not k.startswith("_"))
METRICS = ("messages", "evictions", "reloads", "unique_reloads",
           "mean_span", "p99_span", "mean_reload_pct", "hot_peak",
           "hot_slot_count")


@pytest.mark.parametrize("case", CASES)
def test_bounded_records_bit_exact(case):
    entry = golden_manifest()[case]
    graph, feats = dataset(entry["dataset"])
    cfg = case_config(entry)
    pc = PipelineConfig(hot_budget=cfg["hot_budget"],
                        chunk_budget=cfg["chunk_budget"],
                        eviction=cfg["eviction"], seed=cfg["seed"],
                        hot_slots=cfg["hot_slots"],
                        evict_batch=cfg["evict_batch"], bound_records=True,
                        backend="stable")
    eng = Engine(graph, case_weights(entry), pc)
    h = torch.as_tensor(feats).cuda()
    for l, g in enumerate(entry["layers"]):
        y, m, layer = eng.layer(l, h)
        for f in METRICS:
            assert getattr(m, f) == g[f], (l, f, getattr(m, f), g[f])
        assert digest_array(y.cpu().numpy()) == g["output_sha"], l
        agg = eng.weights.agg_dim(l)
        assert layer.record_bytes() <= max(1, g["hot_slot_count"]) * agg * 4
        w = agg * 4
        # ColdStore byte accounting (oocgnn/memstore.py:52-82)
        assert m.bytes_written == g["evictions"] * w
        assert m.bytes_read == g["reloads"] * w
        h = y
    eng.close()


def test_bounded_records_large_budget_sweep():
    """A 1M-edge graph with a 2 % slot budget: the bounded pass (tcgen05
    backend) equals the unbounded one bit for bit, with ~50 blocks."""
    from paper_2605_09402_b200 import storage as S
    graph, feats = S.synthetic_in_memory("uniform", 100_000, 10, 64, 5)
    w = S.random_weights(S.ModelKind.SAGE, [64, 64, 16], 2)
    outs = []
    for bound in (False, True):
        eng = Engine(graph, w, PipelineConfig(hot_slots=2000,
                                              bound_records=bound,
                                              backend="tcgen05",
                                              transform_first=False))
        y, ms = eng.infer(torch.as_tensor(feats).cuda())
        outs.append((y.cpu().numpy(), [(m.evictions, m.reloads, m.hot_peak)
                                       for m in ms]))
        eng.close()
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1]
