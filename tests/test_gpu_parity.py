"""GPU parity: the sm_100a engine against the reference's golden vectors
(tests/golden, produced by the unmodified reference) and the CPU oracle.

Bar: integer work (messages, evictions, reloads, unique reloads, hot
peak, spans, reload %, victim / reload / graduation logs) bit-exact; with
the ``stable`` transform backend the per-layer embeddings are bit-exact
too (same f32 operation order as the reference engine).
"""

import numpy as np
import pytest
import torch

from helpers import (case_config, case_weights, dataset, digest_array,
                     flatten_events, golden_arrays, golden_manifest, unflatten)
from paper_2605_09402_b200 import _native as N
from paper_2605_09402_b200.chunks import chunk_from_csr, chunk_rows
from paper_2605_09402_b200.errors import (IncompleteLayerError,
                                          StateTransitionError)
from paper_2605_09402_b200.iostats import IOCounters
from paper_2605_09402_b200.orchestrator import (finalize_layer, init_layer,
                                                process_chunk)
from paper_2605_09402_b200.runtime import Engine, PipelineConfig

pytestmark = pytest.mark.gpu

CASES = sorted(k for k in golden_manifest() if not k.startswith("_"))
METRICS = ("messages", "evictions", "reloads", "unique_reloads",
           "mean_span", "p99_span", "mean_reload_pct", "hot_peak",
           "hot_slot_count")


def engine_for(case, **over):
    entry = golden_manifest()[case]
    graph, feats = dataset(entry["dataset"])
    cfg = case_config(entry)
    pc = PipelineConfig(hot_budget=cfg["hot_budget"],
                        chunk_budget=cfg["chunk_budget"],
                        eviction=cfg["eviction"], seed=cfg["seed"],
                        hot_slots=cfg["hot_slots"],
                        evict_batch=cfg["evict_batch"], **over)
    return entry, Engine(graph, case_weights(entry), pc), feats


@pytest.mark.parametrize("case", CASES)
def test_resident_layers_bit_exact(case):
    """run-resident + stable transform: every layer's output, metrics and
    the full integer event log equal the reference's."""
    entry, eng, feats = engine_for(case, record_log=True)
    h = torch.as_tensor(feats).cuda()
    for l, g in enumerate(entry["layers"]):
        y, m, layer = eng.layer(l, h)
        assert digest_array(y.cpu().numpy()) == g["output_sha"], l
        for f in METRICS:
            assert getattr(m, f) == g[f], (l, f, getattr(m, f), g[f])
        assert digest_array(layer.log(N.LOG_VICTIMS)) == g["victims_sha"]
        assert digest_array(layer.log(N.LOG_RELOADS)) == g["reloads_sha"]
        assert digest_array(layer.log(N.LOG_GRADUATED)) == g["graduated_sha"]
        layer.close()
        h = y
    eng.close()


@pytest.mark.parametrize("case", CASES)
def test_resident_fast_path_metrics(case):
    """Without logs the control plane may prove the layer eviction-free
    and answer in closed form; integers must not change."""
    entry, eng, feats = engine_for(case)
    h = torch.as_tensor(feats).cuda()
    for l, g in enumerate(entry["layers"]):
        y, m, layer = eng.layer(l, h)
        layer.close()
        if g["evictions"] == 0 and g["hot_peak"] <= g["hot_slot_count"]:
            pass  # fast path is allowed; exactness checked below either way
        for f in METRICS:
            assert getattr(m, f) == g[f], (l, f, getattr(m, f), g[f])
        assert digest_array(y.cpu().numpy()) == g["output_sha"]
        h = y
    eng.close()


OPERATOR_CASES = [c for c in CASES if golden_manifest()[c]["dataset"]
                  in ("fig2", "small", "half", "uniform")]


@pytest.mark.parametrize("case", OPERATOR_CASES + ["pa_sage_10pct",
                                                   "cfg1_sage"])
@pytest.mark.parametrize("tile_rows", [1, 7, 1000])
def test_streamed_layers_bit_exact(case, tile_rows):
    _streamed_case(case, tile_rows)


TILE_PATH = r"""
import sys
sys.path.insert(0, %r)
sys.path.insert(0, %r)
import test_gpu_parity as T
for case in %r:
    for rows in (7, 1000):
        T._streamed_case(case, rows)
print("ok")
"""


def test_streamed_two_buffer_tile_path_bit_exact():
    """Inputs above ATLAS_STREAM_WHOLE_MAX_BYTES cycle through two tile
    buffers with per-tile aggregation (agg_tile, per-destination cursors);
    forced here on small inputs (fresh process: the limit is read once)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    here = Path(__file__).resolve().parent
    cases = ["small_gcn_tight", "small_sage", "small_gin_tight",
             "half_sage_slots300", "uniform_gin", "pa_sage_10pct"]
    env = dict(os.environ, ATLAS_STREAM_WHOLE_MAX_BYTES="0")
    out = subprocess.run([sys.executable, "-c",
                          TILE_PATH % (str(here.parent), str(here), cases)],
                         env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    assert out.stdout.strip().endswith("ok")


def _streamed_case(case, tile_rows):
    """Host-resident input streamed to HBM in tiles (double-buffered side
    stream): outputs and integers identical to the reference."""
    if tile_rows == 1 and golden_manifest()[case]["dataset"] in ("pa", "cfg1",
                                                                 "uniform"):
        pytest.skip("one-row tiles only on the small graphs")
    entry, eng, feats = engine_for(case)
    h = torch.as_tensor(feats).pin_memory()
    for l, g in enumerate(entry["layers"]):
        eng.config.stream_tile_bytes = tile_rows * h.stride(0) * \
            h.element_size()
        y, m, layer = eng.layer(l, h)
        assert digest_array(y.cpu().numpy()) == g["output_sha"], l
        for f in METRICS:
            assert getattr(m, f) == g[f], (l, f, getattr(m, f), g[f])
        h = y.cpu().pin_memory()
    eng.close()


@pytest.mark.parametrize("case", OPERATOR_CASES)
def test_operator_triple_matches_reference(case):
    """init_layer / process_chunk / finalize_layer on the reference chunk
    plan: the sink sees the reference's graduation order and batching and
    the aggregation rows the reference transform consumed."""
    from oracle import engine as OE

    entry = golden_manifest()[case]
    graph, feats = dataset(entry["dataset"])
    w = case_weights(entry)
    cfg = case_config(entry)
    h = feats
    for l, g in enumerate(entry["layers"]):
        dt = "f16" if h.dtype == np.float16 else "f32"
        rows = chunk_rows(graph.num_vertices, w.embedding_dim(l), dt,
                          cfg["chunk_budget"])
        ctx = init_layer(graph.in_degrees, w, l,
                         hot_budget_bytes=cfg["hot_budget"],
                         io=IOCounters(), eviction=cfg["eviction"],
                         seed=cfg["seed"], hot_slots=cfg["hot_slots"],
                         evict_batch=cfg["evict_batch"])
        batches, agg = [], np.full((graph.num_vertices, w.agg_dim(l)),
                                   np.nan, np.float32)

        class Sink:
            def add_batch(self, vs, r):
                batches.append(np.asarray(vs).tolist())
                agg[vs] = r

        for s in range(0, graph.num_vertices, rows):
            e = min(s + rows, graph.num_vertices)
            process_chunk(ctx, chunk_from_csr(graph, h, s, e), Sink())
        m = finalize_layer(ctx)
        assert digest_array(flatten_events(batches)) == g["graduated_sha"]
        for f in METRICS:
            assert getattr(m, f) == g[f], (l, f, getattr(m, f), g[f])
        out = OE.stable_transform(agg, w.layers[l].weight, w.layers[l].bias,
                                  relu=l < len(w.layers) - 1)
        assert digest_array(out) == g["output_sha"]
        ctx.memory.close()
        h = out


def test_full_arrays_small_cases():
    """Small cases carry full arrays: compare element-wise too."""
    for case in ("small_sage_tight", "fig2_gin"):
        entry, eng, feats = engine_for(case, record_log=True)
        arrays = golden_arrays(case)
        y, metrics = eng.infer(torch.as_tensor(feats).cuda(),
                               keep_layers=True)
        for l, yl in enumerate(eng.last_layers):
            np.testing.assert_array_equal(yl.cpu().numpy(),
                                          arrays[f"L{l}_out"])
        eng.close()


def test_incomplete_layer_detected():
    graph, feats = dataset("fig2")
    from paper_2605_09402_b200.storage import ModelKind, random_weights
    w = random_weights(ModelKind.GCN, [8, 2], 5)
    ctx = init_layer(graph.in_degrees, w, 0, hot_budget_bytes=1 << 20)
    sink = type("S", (), {"add_batch": lambda self, v, r: None})()
    process_chunk(ctx, chunk_from_csr(graph, feats, 0, 2), sink)
    with pytest.raises(IncompleteLayerError):
        finalize_layer(ctx)


def test_completed_vertex_offered_messages_raises():
    graph, feats = dataset("fig2")
    from paper_2605_09402_b200.storage import ModelKind, random_weights
    w = random_weights(ModelKind.GCN, [8, 2], 5)
    ctx = init_layer(graph.in_degrees, w, 0, hot_budget_bytes=1 << 20)
    sink = type("S", (), {"add_batch": lambda self, v, r: None})()
    whole = chunk_from_csr(graph, feats, 0, 6)
    process_chunk(ctx, whole, sink)
    with pytest.raises(StateTransitionError):
        process_chunk(ctx, whole, sink)


def test_stable_transform_bit_exact_vs_reference_backend():
    from oracle import engine as OE
    from paper_2605_09402_b200.compute import MatmulBackend, _apply_device
    rng = np.random.default_rng(0)
    # covers every register-tile width (TN 8/4/3/2), K not a multiple of
    # the 16-wide k tile, unaligned rows (scalar staging), partial row
    # tiles, more rows than one wave of persistent CTAs, and N > 128
    # (the untiled fallback)
    for m, k, n in [(1000, 100, 128), (37, 256, 47), (5, 8, 2), (0, 4, 3),
                    (40961, 100, 128), (4099, 128, 47), (1000, 99, 64),
                    (513, 130, 33), (300, 256, 100), (10, 5, 1),
                    (777, 64, 57), (200, 17, 130)]:
        x = rng.standard_normal((m, k)).astype(np.float32)
        x[rng.random(x.shape) < 0.01] = -0.0
        w = rng.standard_normal((n, k)).astype(np.float32)
        b = rng.standard_normal(n).astype(np.float32)
        b[:: 7] = -0.0
        for relu in (False, True):
            got = _apply_device(MatmulBackend.code, x, w, b, relu=relu)
            want = OE.stable_transform(x, w, b, relu=relu)
            np.testing.assert_array_equal(got.view(np.uint32),
                                          want.view(np.uint32))


@pytest.mark.parametrize("m,k,n,relu", [(1000, 100, 128, True),
                                        (4099, 128, 47, False),
                                        (300, 256, 128, True),
                                        (129, 8, 2, True), (64, 2048, 19, False),
                                        (5000, 128, 256, True),
                                        (100000, 128, 128, False),
                                        (2400, 100, 64, True),
                                        (777, 36, 120, False),
                                        (100000, 256, 128, True),
                                        (50000, 512, 100, False),
                                        # 128 < n <= 192: the streamed-W
                                        # register split with 2 A stages
                                        (30001, 256, 172, True),
                                        (4096, 64, 192, False)])
def test_tcgen05_transform_3xtf32_accuracy(m, k, n, relu):
    """tcgen05 backend: |y - y_f64| <= 2e-6 * (|x| |w| row-col scale)."""
    from paper_2605_09402_b200.compute import Tcgen05Backend
    from paper_2605_09402_b200.storage import LayerWeights
    from paper_2605_09402_b200.compute import transform
    rng = np.random.default_rng(m + k + n)
    x = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    w = (rng.uniform(-1, 1, (n, k)) / np.sqrt(k)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, n).astype(np.float32)
    got = transform(x, LayerWeights(k, n, w, b), apply_activation=relu,
                    backend=Tcgen05Backend())
    ref = x.astype(np.float64) @ w.astype(np.float64).T + b
    if relu:
        ref = np.maximum(ref, 0.0)
    scale = np.abs(x).astype(np.float64) @ np.abs(w).astype(np.float64).T
    err = np.abs(got - ref)
    assert np.all(err <= 4e-6 * (scale + 1e-3)), float((err / (scale + 1e-3)).max())


def test_tiny_and_huge_inputs_take_the_exact_division():
    """Subnormal / tiny / huge inputs: the guarded IEEE division path must
    keep records bit-identical to the reference order of f32 operations."""
    from oracle import engine as OE
    from paper_2605_09402_b200.storage import (ModelKind, random_weights,
                                               synthetic_in_memory)
    graph, feats = synthetic_in_memory("uniform", 3000, 7, 8, 21)
    rng = np.random.default_rng(4)
    pick = rng.random(feats.shape)
    feats = feats.copy()
    feats[pick < 0.05] = np.float32(1e-39)      # subnormal
    feats[(pick > 0.05) & (pick < 0.1)] = np.float32(3e-31)  # tiny normal
    feats[pick > 0.97] = np.float32(3e37)       # huge
    for kind in (ModelKind.GCN, ModelKind.SAGE):
        w = random_weights(kind, [8, 4], 5)
        eng = Engine(graph, w, PipelineConfig(chunk_budget=4096,
                                              hot_slots=3000))
        y, m, _ = eng.layer(0, torch.as_tensor(feats).cuda())
        rows = max(1, 4096 // (8 * 4))
        want, _, _ = OE.run_layer(graph.offsets, graph.neighbors,
                                  graph.in_degrees, feats, int(kind),
                                  w.layers[0].weight, w.layers[0].bias,
                                  relu=False, embed_dim=8,
                                  agg_dim=w.agg_dim(0), chunk_rows=rows,
                                  slot_count=3000)
        np.testing.assert_array_equal(y.cpu().numpy(), want)
        eng.close()


@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("feat_dtype", ["f32", "f16"])
def test_tcgen05_pipeline_within_tolerance(kind, feat_dtype):
    """Whole 3-layer inference with the tcgen05 (3xTF32) transform against
    the float64 gather oracle (oracle/gather.py = oocgnn/oracle.py).
    Stated tolerance, per layer: max |y - y64| <= 1e-5 * max|y64|. The
    reference's own bar is 1e-4 absolute on unit-scale outputs
    (tests/test_acceptance.py:43); GIN's raw sums grow to |y| ~ 420 by layer
    3 here, where the reference's own f32 engine is 1.5e-4 off f64, so the
    bar is stated relative. 3xTF32 keeps ~2^-22 per product; the f32
    pipeline's rounding over three chained layers gives ~3e-6 measured.
    Integer metrics must equal the bit-exact (stable) run's."""
    from oracle import gather as OG
    from paper_2605_09402_b200.storage import (ModelKind, random_weights,
                                               synthetic_in_memory)
    graph, feats = synthetic_in_memory("uniform", 20000, 9, 64, 11)
    if feat_dtype == "f16":
        feats = feats.astype(np.float16)
    w = random_weights(ModelKind(kind), [64, 96, 128, 40], 5, gin_epsilon=0.25)
    want = OG.per_layer(graph.num_vertices, graph.offsets, graph.neighbors,
                        graph.in_degrees, feats.astype(np.float64), kind,
                        [(lw.weight, lw.bias) for lw in w.layers],
                        gin_epsilon=w.gin_epsilon)
    runs = {}
    for backend in ("tcgen05", "stable"):
        eng = Engine(graph, w, PipelineConfig(chunk_budget=1 << 20,
                                              hot_slots=20000,
                                              backend=backend))
        _, metrics = eng.infer(torch.as_tensor(feats).cuda(),
                               keep_layers=True)
        runs[backend] = ([y.double().cpu().numpy() for y in eng.last_layers],
                         metrics)
        eng.close()
    for l, (got, ref) in enumerate(zip(runs["tcgen05"][0], want)):
        err = float(np.abs(got - ref).max())
        assert err <= 1e-5 * float(np.abs(ref).max()), (l, err)
    for a, b in zip(runs["tcgen05"][1], runs["stable"][1]):
        for f in METRICS:
            assert getattr(a, f) == getattr(b, f), f


@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("transform_first", [True, False])
def test_tcgen05_wide_input_transform_first(kind, transform_first):
    """A wide f16 input layer (256 -> 64 -> 24): with transform_first the
    tcgen05 backend aggregates z = h . W^T (f16 input on the tensor cores,
    SAGE's self half added in the fused epilogue); either way every layer
    is within the stated tolerance of the float64 oracle and the integer
    metrics equal the bit-exact run's."""
    from oracle import gather as OG
    from paper_2605_09402_b200.storage import (ModelKind, random_weights,
                                               synthetic_in_memory)
    graph, feats = synthetic_in_memory("uniform", 6000, 7, 256, 21)
    feats = feats.astype(np.float16)
    w = random_weights(ModelKind(kind), [256, 64, 24], 5, gin_epsilon=0.25)
    want = OG.per_layer(graph.num_vertices, graph.offsets, graph.neighbors,
                        graph.in_degrees, feats.astype(np.float64), kind,
                        [(lw.weight, lw.bias) for lw in w.layers],
                        gin_epsilon=w.gin_epsilon)
    runs = {}
    for backend in ("tcgen05", "stable"):
        eng = Engine(graph, w, PipelineConfig(
            chunk_budget=256 << 10, hot_slots=700, backend=backend,
            transform_first=transform_first))
        if backend == "tcgen05":
            assert [eng.transform_first(l) for l in range(2)] == \
                [transform_first, transform_first]
        _, metrics = eng.infer(torch.as_tensor(feats).cuda(),
                               keep_layers=True)
        runs[backend] = ([y.double().cpu().numpy() for y in eng.last_layers],
                         metrics)
        eng.close()
    for l, (got, ref) in enumerate(zip(runs["tcgen05"][0], want)):
        err = float(np.abs(got - ref).max())
        assert err <= 1e-5 * float(np.abs(ref).max()), (l, err)
    for a, b in zip(runs["tcgen05"][1], runs["stable"][1]):
        for f in METRICS:
            assert getattr(a, f) == getattr(b, f), f


def test_topology_refresh_rebinds_layers():
    """Engine.update_graph with a different graph of the same size: the
    cached layers take the new in-degrees from the device graph and the
    result equals a fresh engine's, bit for bit (stable backend)."""
    from paper_2605_09402_b200.storage import (ModelKind, random_weights,
                                               synthetic_in_memory)
    g1, feats = synthetic_in_memory("uniform", 5000, 6, 16, 3)
    g2, _ = synthetic_in_memory("uniform", 5000, 9, 16, 4)
    w = random_weights(ModelKind.SAGE, [16, 12, 8], 5)
    cfg = dict(chunk_budget=32 << 10, hot_slots=300)
    x = torch.as_tensor(feats).cuda()
    eng = Engine(g1, w, PipelineConfig(**cfg))
    eng.infer(x)
    eng.update_graph(g2.offsets, g2.neighbors, g2.in_degrees)
    y, m = eng.infer(x)
    fresh = Engine(g2, w, PipelineConfig(**cfg))
    y2, m2 = fresh.infer(x)
    assert torch.equal(y, y2)
    for a, b in zip(m, m2):
        for f in METRICS:
            assert getattr(a, f) == getattr(b, f), f
    eng.close()
    fresh.close()


@pytest.mark.parametrize("transform_first", [True, False])
def test_host_output_slices(transform_first):
    """infer(..., host_out=pinned): the final output reaches the host
    (sliced D2H behind a transform-first last layer) bit-identical to the
    device result."""
    from paper_2605_09402_b200.storage import (ModelKind, random_weights,
                                               synthetic_in_memory)
    graph, feats = synthetic_in_memory("uniform", 7001, 5, 32, 9)
    w = random_weights(ModelKind.GCN, [32, 16, 6], 5)
    eng = Engine(graph, w, PipelineConfig(backend="tcgen05", hot_slots=7001,
                                          transform_first=transform_first))
    assert eng.transform_first(1) == transform_first
    host = torch.empty((7001, 6), dtype=torch.float32).pin_memory()
    y, _ = eng.infer(torch.as_tensor(feats).pin_memory(), host_out=host)
    torch.cuda.synchronize()
    assert torch.equal(host, y.cpu())
    eng.close()


def test_transform_first_streams_host_input():
    """A pinned-host f16 input of a transform-first layer streams to HBM in
    row tiles, each transformed as it lands: outputs and metrics equal the
    device-resident input's, bit for bit."""
    from paper_2605_09402_b200.storage import (ModelKind, random_weights,
                                               synthetic_in_memory)
    graph, feats = synthetic_in_memory("uniform", 9000, 6, 256, 17)
    feats = feats.astype(np.float16)
    w = random_weights(ModelKind.SAGE, [256, 32, 8], 5)
    cfg = dict(backend="tcgen05", hot_slots=9000, chunk_budget=64 << 10)
    eng = Engine(graph, w, PipelineConfig(stream_tile_bytes=700 * 512, **cfg))
    assert eng.transform_first(0)
    y_host, m_host = eng.infer(torch.as_tensor(feats).pin_memory())
    y_dev, m_dev = eng.infer(torch.as_tensor(feats).cuda())
    assert torch.equal(y_host, y_dev)
    for a, b in zip(m_host, m_dev):
        for f in METRICS:
            assert getattr(a, f) == getattr(b, f), f
    eng.close()


@pytest.mark.parametrize("backend", ["stable", "tcgen05"])
@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("shape", ["no_edges", "one_vertex_loop",
                                   "isolated_hub"])
def test_degenerate_graphs_match_oracle(backend, kind, shape):
    """Edge cases the reference's own tests hold (empty adjacency, a
    single self-looped vertex, zero in-degree next to a 500-in-degree hub):
    the engine's layers equal the reference-pinned oracle (bit-exact with
    the stable backend, 1e-5 relative with tcgen05) with identical metrics."""
    from oracle import engine as OE
    from paper_2605_09402_b200.storage import (ModelKind, edges_to_csr,
                                               random_weights)
    if shape == "no_edges":
        g = edges_to_csr(np.zeros(0, np.int64), np.zeros(0, np.int64), 37)
    elif shape == "one_vertex_loop":
        g = edges_to_csr(np.array([0]), np.array([0]), 1)
    else:
        src = np.concatenate([np.arange(1, 501), np.arange(600, 700)])
        dst = np.concatenate([np.zeros(500, np.int64),
                              np.arange(700, 800)])
        g = edges_to_csr(src, dst, 900)
    v = g.num_vertices
    feats = np.random.default_rng(2).uniform(-1, 1, (v, 16)).astype(
        np.float32)
    w = random_weights(ModelKind(kind), [16, 8, 4], 5, gin_epsilon=0.5)
    eng = Engine(g, w, PipelineConfig(backend=backend, hot_slots=max(1, v),
                                      chunk_budget=512))
    _, metrics = eng.infer(torch.as_tensor(feats).cuda(), keep_layers=True)
    h = feats
    for l, lw in enumerate(w.layers):
        rows = max(1, 512 // (w.embedding_dim(l) * 4))
        want, m, _ = OE.run_layer(g.offsets, g.neighbors, g.in_degrees, h,
                                  kind, lw.weight, lw.bias,
                                  relu=l < len(w.layers) - 1,
                                  embed_dim=w.embedding_dim(l),
                                  agg_dim=w.agg_dim(l), chunk_rows=rows,
                                  slot_count=max(1, v), gin_epsilon=0.5)
        got = eng.last_layers[l].cpu().numpy()
        if backend == "stable":
            np.testing.assert_array_equal(got, want)
        else:
            assert np.abs(got - want).max() <= \
                1e-5 * max(1.0, float(np.abs(want).max()))
        for f in ("messages", "evictions", "reloads", "mean_span",
                  "p99_span", "hot_peak"):
            assert getattr(metrics[l], f) == getattr(m, f), (l, f)
        h = want
    eng.close()


@pytest.mark.parametrize("m,k,n,relu", [(300000, 1024, 128, True),
                                        (5000, 1024, 19, False),
                                        (70000, 128, 128, True),
                                        (1000, 64, 200, False)])
def test_tcgen05_f16_input_transform_accuracy(m, k, n, relu):
    """f16 inputs on kind::f16 (256-row tiles when N <= 128, 128-row tiles
    above): |y - y_f64| <= 4e-6 * (|x| |w| + 1e-3), the 3xTF32 bar."""
    from paper_2605_09402_b200.engine import transform_typed
    g = torch.Generator(device="cuda").manual_seed(m + k + n)
    x = (torch.rand((m, k), device="cuda", generator=g) * 2 - 1).half()
    w = (torch.rand((n, k), device="cuda", generator=g) * 2 - 1) / k ** 0.5
    b = (torch.rand(n, device="cuda", generator=g) - 0.5) * 0.2
    y = torch.empty((m, n), dtype=torch.float32, device="cuda")
    transform_typed(x, w, b, relu, y, N.BACKEND_TCGEN05)
    ref = x.double() @ w.double().T + b.double()
    if relu:
        ref = ref.clamp_min(0.0)
    scale = x.double().abs() @ w.double().abs().T
    err = (y.double() - ref).abs()
    assert bool((err <= 4e-6 * (scale + 1e-3)).all()), \
        float((err / (scale + 1e-3)).max())


@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("out", [3, 13, 19, 24, 30, 47, 52, 60])
def test_transform_first_narrow_widths(kind, out):
    """Every lanes-per-row x chunks-per-lane shape of the narrow
    transform-first aggregation (agg_tf_multi: 1..16 chunks of z per row,
    cfg2's 47-wide last layer = 12 chunks on 4 lanes x 3) against the
    float64 oracle, same stated tolerance as the pipeline test."""
    from oracle import gather as OG
    from paper_2605_09402_b200.storage import (ModelKind, random_weights,
                                               synthetic_in_memory)
    graph, feats = synthetic_in_memory("pa", 5000, 11, 64, 3 + out)
    w = random_weights(ModelKind(kind), [64, out], 5, gin_epsilon=0.25)
    want = OG.per_layer(graph.num_vertices, graph.offsets, graph.neighbors,
                        graph.in_degrees, feats.astype(np.float64), kind,
                        [(lw.weight, lw.bias) for lw in w.layers],
                        gin_epsilon=w.gin_epsilon)
    eng = Engine(graph, w, PipelineConfig(chunk_budget=1 << 20,
                                          hot_slots=5000, backend="tcgen05",
                                          transform_first=True))
    assert eng.transform_first(0)
    _, _ = eng.infer(torch.as_tensor(feats).cuda(), keep_layers=True)
    got = eng.last_layers[0].double().cpu().numpy()
    eng.close()
    err = float(np.abs(got - want[0]).max())
    assert err <= 1e-5 * float(np.abs(want[0]).max()), err


def test_user_host_backend_plugin_matches_stable():
    """A user MatmulBackend object without a device code (the reference's
    plug-in protocol: name, max_batch_rows, apply(batch, weight, bias)) is
    honoured on the host, exactly as oocgnn/compute.py:76-97 calls it; the
    aggregation stays on the device. It is never a fallback: the built-in
    backends always carry a device code. Written as the reference's own
    f32 chain (out = b; out += x_k * w_k, k ascending), it reproduces the
    stable backend's bits."""
    from paper_2605_09402_b200 import _native as NN
    from paper_2605_09402_b200.storage import (ModelKind, random_weights,
                                               synthetic_in_memory)

    class ChainBackend:
        name = "user_chain"
        max_batch_rows = 1000

        def __init__(self):
            self.calls = 0

        def apply(self, batch, weight, bias):
            self.calls += 1
            out = np.broadcast_to(bias.astype(np.float32),
                                  (len(batch), len(bias))).copy()
            for k in range(batch.shape[1]):
                out += batch[:, k:k + 1] * weight[:, k]
            return out

    graph, feats = synthetic_in_memory("pa", 3000, 7, 24, 17)
    w = random_weights(ModelKind.SAGE, [24, 16, 8], 5)
    user = ChainBackend()
    lib = NN.load_library()
    outs = {}
    for name, be in (("stable", "stable"), ("user", user)):
        eng = Engine(graph, w, PipelineConfig(chunk_budget=64 << 10,
                                              hot_slots=3000, backend=be))
        before = lib.atlas_kernel_launches()
        y, _ = eng.infer(torch.as_tensor(feats).cuda())
        torch.cuda.synchronize()
        assert lib.atlas_kernel_launches() > before  # device aggregation
        outs[name] = y.cpu().numpy()
        eng.close()
    assert user.calls >= 6  # 3000 rows in batches of 1000, two layers
    np.testing.assert_array_equal(outs["user"], outs["stable"])


@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("embed", ["f16", "bf16"])
@pytest.mark.parametrize("transform_first", [True, False])
def test_two_byte_embeddings_within_tolerance(kind, embed, transform_first):
    """Intermediate embeddings stored in f16 / bf16 (PipelineConfig.
    embed_dtype, the slice workloads' default): 2-byte rows through the
    aggregation kernels (widened exactly, f32 accumulation) and 2-byte
    transform inputs (kind::f16 for f16, tf32 for bf16). Stated tolerance
    per layer against the float64 oracle: 3e-3 * max|y| for f16, 2e-2 for
    bf16 (one rounding of each stored embedding: 2^-11 / 2^-8 relative,
    compounded over the layers); integer metrics equal the f32 run's."""
    from oracle import gather as OG
    from paper_2605_09402_b200.storage import (ModelKind, random_weights,
                                               synthetic_in_memory)
    graph, feats = synthetic_in_memory("pa", 8000, 9, 64, 29)
    w = random_weights(ModelKind(kind), [64, 96, 128, 40], 5, gin_epsilon=0.25)
    want = OG.per_layer(graph.num_vertices, graph.offsets, graph.neighbors,
                        graph.in_degrees, feats.astype(np.float64), kind,
                        [(lw.weight, lw.bias) for lw in w.layers],
                        gin_epsilon=w.gin_epsilon)
    tol = {"f16": 3e-3, "bf16": 2e-2}[embed]
    runs = {}
    for dt in (embed, "f32"):
        eng = Engine(graph, w, PipelineConfig(
            chunk_budget=256 << 10, hot_slots=8000, backend="tcgen05",
            embed_dtype=dt, transform_first=transform_first))
        _, metrics = eng.infer(torch.as_tensor(feats).cuda(),
                               keep_layers=True)
        runs[dt] = ([y.double().cpu().numpy() for y in eng.last_layers],
                    metrics)
        eng.close()
    for l, (got, ref) in enumerate(zip(runs[embed][0], want)):
        err = float(np.abs(got - ref).max())
        assert err <= tol * float(np.abs(ref).max()), (l, err)
    for a, b in zip(runs[embed][1], runs["f32"][1]):
        for f in METRICS:
            assert getattr(a, f) == getattr(b, f), f
