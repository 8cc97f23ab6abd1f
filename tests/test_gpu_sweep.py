"""The sweep replay (csrc/sweep.cu) against the per-element machine
(csrc/engine.cu) on graphs far larger than the golden cases, under eviction
pressure: every integer metric, the per-chunk reload / touched counters and
the output must be identical. The per-element machine is itself pinned to
the reference's event logs (tests/test_gpu_parity.py); the golden cases run
through the sweep in test_resident_fast_path_metrics."""

import os

import numpy as np
import pytest
import torch

from helpers import digest_array
from paper_2605_09402_b200 import storage as S
from paper_2605_09402_b200.runtime import Engine, PipelineConfig

pytestmark = pytest.mark.gpu

FIELDS = ("messages", "evictions", "reloads", "unique_reloads", "mean_span",
          "p99_span", "mean_reload_pct", "hot_peak", "hot_slot_count")

CASES = [
    # kind, V, deg, dim, model, hot fraction, policy, chunk budget
    ("uniform", 200_000, 10, 32, "GCN", 0.05, "minpend", 1 << 20),
    ("pa", 150_000, 8, 32, "SAGE", 0.08, "minpend", 1 << 20),
    ("uniform", 120_000, 12, 16, "GIN", 0.10, "minpend", 256 << 10),
    ("uniform", 150_000, 6, 32, "SAGE", 0.05, "lru", 512 << 10),
    ("pa", 100_000, 10, 32, "GCN", 0.03, "lru", 1 << 20),
    ("uniform", 60_000, 4, 64, "GCN", 0.002, "minpend", 64 << 10),
]


def run(kind, v, deg, dim, model, frac, policy, budget, sweep, coop=True):
    os.environ["ATLAS_SWEEP"] = "1" if sweep else "0"
    os.environ["ATLAS_SWEEP_COOP"] = "1" if coop else "0"
    try:
        graph, feats = S.synthetic_in_memory(kind, v, deg, dim, 11)
        w = S.random_weights(S.ModelKind[model], [dim, 16, 8], 3)
        cfg = PipelineConfig(chunk_budget=budget, eviction=policy,
                             hot_slots=max(1, int(v * frac)),
                             force_exact=True, backend="stable")
        eng = Engine(graph, w, cfg)
        h = torch.as_tensor(feats).cuda()
        out = []
        for l in range(len(w.layers)):
            y, m, layer = eng.layer(l, h)
            rel, tou = layer.chunk_stats()
            out.append(({f: getattr(m, f) for f in FIELDS}, rel.tolist(),
                        tou.tolist(), digest_array(y.cpu().numpy())))
            h = y
        eng.close()
        return out
    finally:
        os.environ.pop("ATLAS_SWEEP", None)
        os.environ.pop("ATLAS_SWEEP_COOP", None)


@pytest.mark.parametrize("case", CASES, ids=[
    f"{c[0]}-{c[4]}-{c[6]}-{c[5]}" for c in CASES])
def test_sweep_equals_per_element_machine(case):
    """Both sweeps (the cooperative grid and the single CTA) against the
    per-element machine."""
    b = run(*case, sweep=False)
    assert sum(layer[0]["evictions"] for layer in b) > 0
    for coop in (True, False):
        a = run(*case, sweep=True, coop=coop)
        for l, (x, y) in enumerate(zip(a, b)):
            assert x[0] == y[0], (coop, l, x[0], y[0])
            assert x[1] == y[1], (coop, l)
            assert x[2] == y[2], (coop, l)
            assert x[3] == y[3], (coop, l)
