"""Small end-to-end workload for compute-sanitizer runs (memcheck,
racecheck, synccheck, initcheck) over every kernel family of the library:

* the cooperative exact control engine with logs (eviction-heavy golden
  cases: victims, reloads, radix-select grid jobs; forced onto the grid
  path with ATLAS_ENGINE_GRID_MIN=1 by the caller if wanted);
* the bit-exact ring aggregation kernels (agg_ring / agg_sub_ring /
  agg_bulk) and the stable transform;
* the sweep replay (csrc/sweep.cu) and the bounded-record blocked pass;
* the tcgen05 transform (3xTF32 register split and f16 hi/lo) and
  transform-first fused passes;
* the streamed K1 path (suffix ring + agg_tile), the operator (per-chunk)
  path, GAT pass A/B.

Every run is also checked against the reference's golden digests, so a
sanitizer pass is a correctness pass too.

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py
"""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from helpers import (case_weights, dataset, digest_array,  # noqa: E402
                     golden_manifest)
from paper_2605_09402_b200 import _native as N  # noqa: E402
from paper_2605_09402_b200.runtime import Engine, PipelineConfig  # noqa: E402

CASES = ["small_gcn_tight", "small_sage_tight", "small_gin_tight",
         "half_sage_slots300", "wide_gcn", "uniform_gin_slots500"]


def config(entry, **kw):
    cfg = dict(entry["config"])
    keep = {k: cfg[k] for k in ("hot_budget", "chunk_budget", "eviction",
                                "seed", "hot_slots", "evict_batch")
            if k in cfg}
    return PipelineConfig(**keep, **kw)


def run_case(case):
    entry = golden_manifest()[case]
    graph, feats = dataset(entry["dataset"])
    w = case_weights(entry)
    # exact engine with logs, stable transform: bit-exact
    eng = Engine(graph, w, config(entry, backend="stable", record_log=True))
    h = torch.as_tensor(feats).cuda()
    for l, g in enumerate(entry["layers"]):
        y, m, layer = eng.layer(l, h)
        assert digest_array(y.cpu().numpy()) == g["output_sha"], (case, l)
        assert digest_array(layer.log(N.LOG_VICTIMS)) == g["victims_sha"]
        layer.close()
        h = y
    eng.close()
    # streamed from pinned host in small tiles
    eng = Engine(graph, w, config(entry, backend="stable",
                                  stream_tile_bytes=16 << 10))
    y, _ = eng.infer(torch.as_tensor(feats).pin_memory())
    assert digest_array(y.cpu().numpy()) == entry["layers"][-1]["output_sha"]
    eng.close()
    # sweep replay (no logs, exact control plane forced) + bounded records
    eng = Engine(graph, w, config(entry, backend="stable", force_exact=True,
                                  bound_records=True))
    y, metrics = eng.infer(torch.as_tensor(feats).cuda())
    assert digest_array(y.cpu().numpy()) == entry["layers"][-1]["output_sha"]
    assert [m.reloads for m in metrics] == \
        [g["reloads"] for g in entry["layers"]]
    eng.close()
    # tcgen05 backend (transform-first where it narrows)
    eng = Engine(graph, w, config(entry, backend="tcgen05"))
    y, metrics = eng.infer(torch.as_tensor(feats).cuda())
    assert [m.evictions for m in metrics] == \
        [g["evictions"] for g in entry["layers"]]
    eng.close()


def run_gat():
    from oracle import gat as OG
    from paper_2605_09402_b200 import storage as S
    from paper_2605_09402_b200.gat import GATEngine, random_gat_weights
    g, _ = S.synthetic_in_memory("uniform", 3000, 8, 4, 4)
    w = random_gat_weights([64, 128, 19], 4, seed=5)
    x = np.random.default_rng(3).uniform(-1, 1, (3000, 64)).astype(
        np.float16)
    want = OG.gat_per_layer(g.offsets, g.neighbors, x.astype(np.float64),
                            w.oracle_layers())
    for zt in ("f32", "f16"):
        eng = GATEngine(g, w, PipelineConfig(backend="tcgen05",
                                             embed_dtype=zt,
                                             chunk_budget=16 << 10,
                                             hot_slots=400))
        y, _ = eng.infer(torch.as_tensor(x).cuda())
        err = np.abs(y.double().cpu().numpy() - want[-1]).max()
        assert err <= 3e-3 * np.abs(want[-1]).max(), err
        eng.close()


def run_extra():
    """Round-2b kernels: the wide streamed-W transform (128 < N <= 192),
    2-byte intermediate embeddings (agg_tf_multi / 2-byte rings)."""
    from paper_2605_09402_b200 import storage as S
    from paper_2605_09402_b200.engine import transform_typed
    x = torch.randn(3001, 256, device="cuda")
    wt = torch.randn(172, 256, device="cuda") / 16
    b = torch.randn(172, device="cuda")
    y = torch.empty(3001, 172, device="cuda")
    transform_typed(x, wt, b, True, y, 1)
    ref = (x.double() @ wt.double().T + b.double()).clamp_min(0)
    assert float((y.double() - ref).abs().max()) < 1e-4
    graph, feats = S.synthetic_in_memory("pa", 4000, 7, 48, 3)
    w = S.random_weights(S.ModelKind.GCN, [48, 64, 20], 5)
    for dt in ("f16", "bf16"):
        eng = Engine(graph, w, PipelineConfig(chunk_budget=64 << 10,
                                              hot_slots=4000,
                                              backend="tcgen05",
                                              embed_dtype=dt))
        eng.infer(torch.as_tensor(feats).cuda())
        eng.close()


def run_operator():
    from paper_2605_09402_b200.chunks import chunk_from_csr, chunk_rows
    from paper_2605_09402_b200.orchestrator import (finalize_layer,
                                                    init_layer,
                                                    process_chunk)
    entry = golden_manifest()["small_sage_tight"]
    graph, feats = dataset(entry["dataset"])
    w = case_weights(entry)

    class Sink:
        def add_batch(self, ids, rows):
            pass

    ctx = init_layer(graph.in_degrees, w, 0, hot_budget_bytes=1 << 20,
                     hot_slots=32)
    rows = chunk_rows(graph.num_vertices, w.embedding_dim(0), "f32", 4096)
    for s in range(0, graph.num_vertices, rows):
        process_chunk(ctx, chunk_from_csr(graph, feats, s,
                                          min(s + rows, graph.num_vertices)),
                      Sink())
    m = finalize_layer(ctx)
    assert m.evictions == entry["layers"][0]["evictions"]
    ctx.memory.close()


if __name__ == "__main__":
    import os
    # racecheck instruments every shared-memory access: the quick probe
    # keeps one case of each model (SANITIZE_QUICK=1)
    quick = os.environ.get("SANITIZE_QUICK") == "1"
    for c in (CASES[:3] if quick else CASES):
        run_case(c)
    run_gat()
    run_extra()
    run_operator()
    torch.cuda.synchronize()
    print("sanitize probe ok", flush=True)
