"""GAT on the GPU (pass A on tcgen05 + fused edge-softmax aggregation)
against the float64 oracle (oracle/gat.py; parity unpinned: the reference
has no GAT). Stated tolerance, per layer:
  z stored f32:  max |y - y64| <= 2e-5 * max |y64|
  z stored f16:  max |y - y64| <= 3e-3 * max |y64|
Integer metrics must equal the GCN control plane's (pending = in-degree,
SURVEY.md A.5) on the same chunk plan and slot budget."""

import numpy as np
import pytest
import torch

from oracle import engine as OE
from oracle import gat as OG
from paper_2605_09402_b200 import gat as G
from paper_2605_09402_b200 import storage as S
from paper_2605_09402_b200.runtime import PipelineConfig

pytestmark = pytest.mark.gpu

TOL = {"f32": 2e-5, "f16": 3e-3, "bf16": 2e-2}


def hub_graph(v=3000, seed=4):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, v, 8 * v)
    dst = rng.integers(50, v, 8 * v)           # 0..49: zero in-degree
    src = np.concatenate([src, np.arange(300), [77, 78]])
    dst = np.concatenate([dst, np.full(300, 60), [77, 78]])  # hub, loops
    return S.edges_to_csr(src, dst, v)


@pytest.mark.parametrize("zdtype", ["f32", "f16"])
@pytest.mark.parametrize("feat_dtype", ["f32", "f16"])
@pytest.mark.parametrize("heads,dims", [(4, [64, 128, 128, 19]),
                                        (2, [24, 16, 5]), (1, [16, 8, 8]),
                                        (1, [16, 100, 12])])
def test_gat_matches_f64_oracle(zdtype, feat_dtype, heads, dims):
    g = hub_graph()
    w = G.random_gat_weights(dims, heads, seed=5)
    x = np.random.default_rng(3).uniform(-1, 1, (g.num_vertices, dims[0]))
    x = x.astype(np.float16 if feat_dtype == "f16" else np.float32)
    want = OG.gat_per_layer(g.offsets, g.neighbors, x.astype(np.float64),
                            w.oracle_layers())
    eng = G.GATEngine(g, w, PipelineConfig(backend="tcgen05",
                                           embed_dtype=zdtype,
                                           chunk_budget=16 << 10,
                                           hot_slots=400))
    _, metrics = eng.infer(torch.as_tensor(x).cuda(), keep_layers=True)
    for l, (y, ref) in enumerate(zip(eng.last_layers, want)):
        got = y.double().cpu().numpy()
        err = float(np.abs(got - ref).max())
        assert err <= TOL[zdtype] * float(np.abs(ref).max()), (l, err)
    # control plane: GCN rules on the layer input's chunk plan (in_dim
    # rows; the dataset dtype at layer 0, f32 afterwards) -- independent of
    # the z storage dtype and padding
    for l, (m, lw) in enumerate(zip(metrics, w.layers)):
        item = 2 if (l == 0 and feat_dtype == "f16") else 4
        rows = max(1, (16 << 10) // (lw.in_dim * item))
        _, om, _ = OE.run_layer(
            g.offsets, g.neighbors, g.in_degrees,
            np.zeros((g.num_vertices, 1), np.float32), OE.GCN,
            np.zeros((1, 1), np.float32), np.zeros(1, np.float32),
            relu=False, embed_dim=1, agg_dim=1, chunk_rows=rows,
            slot_count=400)
        for f in ("messages", "evictions", "reloads", "unique_reloads",
                  "mean_span", "p99_span", "hot_peak"):
            assert getattr(m, f) == getattr(om, f), (l, f)
    eng.close()


def test_gat_single_vertex_and_empty_range():
    """1-vertex graph with a self loop, and a graph without edges."""
    for src, dst, v in (([0], [0], 1), ([], [], 5)):
        g = S.edges_to_csr(np.array(src, np.int64), np.array(dst, np.int64),
                           v)
        w = G.random_gat_weights([8, 8, 3], 2, seed=1)
        x = np.random.default_rng(0).uniform(-1, 1, (v, 8)).astype(np.float32)
        want = OG.gat_per_layer(g.offsets, g.neighbors, x, w.oracle_layers())
        eng = G.GATEngine(g, w, PipelineConfig(backend="tcgen05"))
        y, _ = eng.infer(torch.as_tensor(x).cuda())
        np.testing.assert_allclose(y.cpu().numpy(), want[-1], atol=1e-5)
        eng.close()
