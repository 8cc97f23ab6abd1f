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
                                        (1, [16, 100, 12]),
                                        # er fused into pass A's epilogue
                                        # (16-column heads, 2 and 8 heads)
                                        (2, [32, 32, 16]),
                                        (8, [64, 128, 8])])
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


@pytest.mark.parametrize("feat_dtype", ["f32", "f16"])
def test_gat_fused_er_equals_extended_weight(feat_dtype):
    """atlas_transform_er (z GEMM on the register-split / f16 kernels with
    er from the epilogue) against pass A through W_ext (el and er as extra
    GEMM rows): z and er equal to f32 rounding (the kernels may order the
    split products differently)."""
    from paper_2605_09402_b200.engine import transform_er, transform_typed
    w = G.random_gat_weights([256, 128, 19], 4, seed=9)
    lw = w.layers[0]
    lay = G.ZLayout(lw.heads, lw.head_dim, 4)
    assert lay.line_rows and lay.el_col == 128
    ext = torch.as_tensor(G.extended_weight(lw, lay)).cuda()
    x = torch.randn(70001, 256, device="cuda")
    if feat_dtype == "f16":
        x = x.half()
    zb = torch.zeros(lay.ncols, device="cuda")
    y_ext = torch.zeros(x.shape[0], lay.ldz, device="cuda")
    transform_typed(x, ext, zb, False, y_ext[:, :lay.ncols], 1)
    ar = np.zeros((lw.heads, lay.head_stride), np.float32)
    ar[:, :lw.head_dim] = lw.attn_r
    y_er = torch.zeros_like(y_ext)
    transform_er(x, ext[:lay.el_col].contiguous(), zb, y_er, lay.el_col,
                 torch.as_tensor(ar.reshape(-1)).cuda(), lay.er_col,
                 lw.heads, lay.head_stride)
    torch.cuda.synchronize()
    a, b = y_ext.cpu().numpy(), y_er.cpu().numpy()
    # different kernels (n = 136 vs 128) may order the split products
    # differently: equal to f32 rounding
    zs = float(np.abs(a[:, :128]).max())
    assert float(np.abs(a[:, :128] - b[:, :128]).max()) <= 2e-6 * zs
    er_a = a[:, lay.er_col:lay.er_col + lw.heads]
    er_b = b[:, lay.er_col:lay.er_col + lw.heads]
    scale = float(np.abs(er_a).max())
    assert float(np.abs(er_a - er_b).max()) <= 2e-5 * scale

