"""Regenerate tests/golden/*.json|npz by running the UNMODIFIED reference.

Run here (the container holding /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``oocgnn`` read-only from /root/reference/pkg/src, runs
``run_inference`` and the ``init_layer/process_chunk/finalize_layer``
operator triple on the cases below, and records:

* per-layer engine outputs (full arrays for small cases, sha256 otherwise);
* per-layer metrics (every CSV column except wall time, plus hot_peak);
* the integer event log: victims of every eviction, every reload batch and
  every graduation batch, captured by wrapping the reference's policy,
  ``MemoryManager._reload_batch`` and ``orchestrator._graduate``;
* the reference's float64 ``oracle_inference`` output.

The GPU box has no /root/reference, so these files are what the GPU
parity tests compare against.
"""

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import oocgnn.memstore as mem  # noqa: E402
import oocgnn.orchestrator as orch  # noqa: E402
import oocgnn.runtime as rt  # noqa: E402
from oocgnn.iostats import IOCounters  # noqa: E402
from oocgnn.chunks import Chunk, plan_chunks  # noqa: E402
from oocgnn.oracle import oracle_inference  # noqa: E402
from oocgnn.storage import (  # noqa: E402
    ModelKind, edges_to_csr, generate_synthetic, load_layer_matrix,
    random_weights, read_csr, write_csr, write_matrix_as_layer)

OUT = Path(__file__).resolve().parent


def digest_array(a) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(str(a.dtype).encode() + str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def flatten_events(events) -> np.ndarray:
    """[[a,b],[c]] -> int64 [2,a,b,1,c]."""
    out = []
    for ev in events:
        out.append(len(ev))
        out.extend(int(x) for x in ev)
    return np.asarray(out, dtype=np.int64)


class Recorder:
    """Wraps the reference's hooks; one log per layer."""

    def __init__(self):
        self.layers = []

    def new_layer(self):
        self.layers.append({"victims": [], "reloads": [], "graduated": []})

    @property
    def cur(self):
        return self.layers[-1]


REC = Recorder()
_make_policy = mem.make_policy
_reload = mem.MemoryManager._reload_batch
_graduate = orch._graduate
_run_layer = rt.run_layer


def traced_make_policy(name, max_pending, seed):
    pol = _make_policy(name, max_pending, seed)
    choose = pol.choose_victims

    def wrapped(k):
        got = choose(k)
        REC.cur["victims"].append(list(got))
        return got
    pol.choose_victims = wrapped
    return pol


def traced_reload(self, vertices):
    REC.cur["reloads"].append(np.asarray(vertices).tolist())
    return _reload(self, vertices)


def traced_graduate(ctx, vertices, sink):
    REC.cur["graduated"].append(np.asarray(vertices).tolist())
    return _graduate(ctx, vertices, sink)


def traced_run_layer(*a, **k):
    REC.new_layer()
    return _run_layer(*a, **k)


mem.make_policy = traced_make_policy
orch.make_policy = traced_make_policy
mem.MemoryManager._reload_batch = traced_reload
orch._graduate = traced_graduate
rt.run_layer = traced_run_layer


METRIC_FIELDS = ["messages", "evictions", "reloads", "unique_reloads",
                 "mean_span", "p99_span", "mean_reload_pct", "hot_peak",
                 "hot_slot_count"]


def metrics_rows(path):
    """metrics.csv as written by the reference (oocgnn/runtime.py:98-111),
    minus the wall_seconds column (timing)."""
    import csv
    with open(path, newline="") as f:
        rows = list(csv.reader(f))
    return [r[:-1] for r in rows]


def dir_digest(layer_dir):
    """sha256 over the sorted (relative path, bytes) of a layer directory,
    plus its file count and total bytes."""
    layer_dir = Path(layer_dir)
    h = hashlib.sha256()
    n = total = 0
    for p in sorted(q for q in layer_dir.rglob("*") if q.is_file()):
        data = p.read_bytes()
        h.update(str(p.relative_to(layer_dir)).encode() + b"\0")
        h.update(data)
        n += 1
        total += len(data)
    return {"sha": h.hexdigest(), "files": n, "bytes": total}


def fig2_dataset(root):
    edges = [(0, 1), (0, 3), (2, 3), (4, 1), (4, 3)]
    g = edges_to_csr(np.array([e[0] for e in edges]),
                     np.array([e[1] for e in edges]), 6)
    feats = np.random.default_rng(3).uniform(-1, 1, (6, 8)).astype(np.float32)
    d = root / "fig2"
    write_csr(g, d)
    write_matrix_as_layer(d / "features", feats)
    return d


DATASETS = {
    # name: (kind, V, degree, dim, seed, dtype)
    "small": ("uniform", 2000, 6, 8, 3, "f32"),
    "uniform": ("uniform", 10_000, 10, 32, 7, "f32"),
    "pa": ("pa", 100_000, 10, 64, 12, "f32"),
    "cfg1": ("uniform", 100_000, 10, 128, 7, "f32"),
    "half": ("uniform", 4000, 8, 16, 11, "f16"),
    # wide rows (the IGB-shaped 1024-d f16 path: bulk-copy aggregation)
    "wide": ("uniform", 3000, 8, 1024, 13, "f16"),
}

SMALL_CFG = dict(hot_budget=1 << 20, chunk_budget=64 << 10,
                 graduation_budget=256 << 10, spill_buffer=256 << 10,
                 partitions=3, queue_capacity=4)

# (case id, dataset, model, dims, weight seed, eps, gain, config, full)
CASES = []
for kind in ModelKind:
    eps = 0.1 if kind == ModelKind.GIN else 0.0
    gain = 0.15 if kind == ModelKind.GIN else 1.0
    CASES.append((f"fig2_{kind.cli_name}", "fig2", kind, [8, 4, 2], 5, eps,
                  gain, {}, True))
    CASES.append((f"small_{kind.cli_name}", "small", kind, [8, 4, 2], 5, eps,
                  1.0, dict(SMALL_CFG), True))
    CASES.append((f"small_{kind.cli_name}_tight", "small", kind, [8, 4, 2],
                  5, eps, 1.0, dict(SMALL_CFG, chunk_budget=4096,
                                    hot_slots=32), True))
    CASES.append((f"uniform_{kind.cli_name}", "uniform", kind, [32, 16, 8],
                  5, eps, gain, {}, False))
    CASES.append((f"uniform_{kind.cli_name}_slots500", "uniform", kind,
                  [32, 16, 8], 5, eps, gain,
                  dict(hot_slots=500, chunk_budget=4096 * 32 * 4), False))
    CASES.append((f"half_{kind.cli_name}_slots300", "half", kind,
                  [16, 8, 4], 5, eps, gain,
                  dict(hot_slots=300, chunk_budget=16 << 10), False))
    CASES.append((f"wide_{kind.cli_name}", "wide", kind, [1024, 600, 16], 5,
                  eps, gain, dict(hot_slots=400, chunk_budget=256 << 10),
                  False))
for pol in ("minpend", "lru", "rnd"):
    CASES.append((f"pa_gcn_{pol}_5pct", "pa", ModelKind.GCN, [64, 32, 16], 5,
                  0.0, 1.0, dict(hot_slots=5000, eviction=pol, seed=1), False))
CASES.append(("pa_sage_10pct", "pa", ModelKind.SAGE, [64, 32, 16], 5, 0.0,
              1.0, dict(hot_slots=10_000), False))
CASES.append(("cfg1_sage", "cfg1", ModelKind.SAGE, [128, 128, 128], 5, 0.0,
              1.0, dict(chunk_budget=64 << 20, hot_slots=100_000), False))
CASES.append(("cfg1_sage_10pct", "cfg1", ModelKind.SAGE, [128, 128, 128], 5,
              0.0, 1.0, dict(chunk_budget=1 << 20, hot_slots=10_000), False))


def main(only=None):
    work = Path(tempfile.mkdtemp(prefix="golden_"))
    ds_dirs = {"fig2": fig2_dataset(work)}
    manifest = {}
    for case, ds, kind, dims, wseed, eps, gain, cfg, full in CASES:
        if only and case not in only:
            continue
        if ds not in ds_dirs:
            gk, v, deg, dim, seed, dt = DATASETS[ds]
            ds_dirs[ds] = work / ds
            generate_synthetic(gk, v, deg, dim, seed, ds_dirs[ds], dtype=dt)
        weights = random_weights(kind, dims, wseed, gin_epsilon=eps,
                                 gain=gain)
        REC.layers.clear()
        out = work / f"run_{case}"
        report = rt.run_inference(ds_dirs[ds], weights,
                                  rt.PipelineConfig(**cfg), out)
        graph = read_csr(ds_dirs[ds])
        feats = load_layer_matrix(ds_dirs[ds] / "features")
        ref64 = oracle_inference(graph, feats, weights, memory_cap=16 << 30)
        entry = {"dataset": ds, "model": int(kind), "dims": dims,
                 "weight_seed": wseed, "gin_epsilon": eps, "gain": gain,
                 "config": cfg, "layers": []}
        arrays = {}
        for l, m in enumerate(report.layers):
            y = load_layer_matrix(out / f"layer_{l}")
            log = REC.layers[l]
            lay = {f: getattr(m, f) for f in METRIC_FIELDS}
            lay["output_sha"] = digest_array(y)
            for key in ("victims", "reloads", "graduated"):
                flat = flatten_events(log[key])
                lay[f"{key}_sha"] = digest_array(flat)
                lay[f"{key}_events"] = len(log[key])
                if full:
                    arrays[f"L{l}_{key}"] = flat
            if full:
                arrays[f"L{l}_out"] = y
            entry["layers"].append(lay)
        entry["metrics_csv"] = metrics_rows(out / "metrics.csv")
        entry["layer_dirs"] = [dir_digest(out / f"layer_{l}")
                               for l in range(len(report.layers))]
        entry["oracle64_sha"] = digest_array(ref64)
        arrays["oracle64"] = ref64 if full else ref64[:64]
        entry["oracle64_absmax"] = float(np.abs(ref64).max())
        manifest[case] = entry
        np.savez_compressed(OUT / f"{case}.npz", **arrays)
        print(case, [(l["messages"], l["evictions"], l["reloads"])
                     for l in entry["layers"]], flush=True)
    # operator-triple chunk plans (oocgnn/chunks.py:36-48)
    plans = {f"{v}_{d}_{t}_{b}": plan_chunks(v, d, t, b) for v, d, t, b in
             [(10, 4, "f32", 64), (10, 4, "f16", 64), (7, 3, "f32", 1),
              (0, 8, "f32", 64), (2_400_000, 100, "f32", 8 << 20),
              (2_400_000, 128, "f32", 8 << 20)]}
    manifest["_plans"] = {k: [len(p), p[:3], p[-1:]] for k, p in plans.items()}
    manifest["_datasets"] = DATASETS
    path = OUT / "golden.json"
    old = json.loads(path.read_text()) if (only and path.exists()) else {}
    old.update(manifest)
    path.write_text(json.dumps(old, indent=1, sort_keys=True))


# --- benchmark-scale case (BASELINE configs[1] = cfg2) -------------------
# One reference run at the headline configuration: 3-layer GCN
# [100,128,128,47] on the uniform V=2.4M / E=62,399,647 graph (seed 7),
# 8 MiB chunks (115 at layer 1), hot_slots = V. ~20 min on one core here.
# Stored in its own manifest (golden_scale.json) so the per-case parity
# suites do not pick it up: per-layer output sha256 and metrics, the
# graduation log digest, metrics.csv, the layer-dir digests, and the
# reference oracle (oocgnn/oracle.py:26-55) per layer on SAMPLE_ROWS
# sampled rows (the truncated model l+1 layers deep, ReLU applied on
# hidden layers as the full model does) with each layer's max |y|.
SCALE_DATASETS = {"cfg2": ("uniform", 2_400_000, 26, 100, 7, "f32")}
SCALE_CASES = [("cfg2_gcn", "cfg2", ModelKind.GCN, [100, 128, 128, 47], 5,
                0.0, 1.0, dict(hot_slots=2_400_000))]
SAMPLE_ROWS = 2048


def scale_goldens():
    from oocgnn.storage import ModelWeights
    work = Path(tempfile.mkdtemp(prefix="golden_scale_"))
    path = OUT / "golden_scale.json"
    manifest = json.loads(path.read_text()) if path.exists() else {}
    for case, ds, kind, dims, wseed, eps, gain, cfg in SCALE_CASES:
        gk, v, deg, dim, seed, dt = SCALE_DATASETS[ds]
        dsdir = work / ds
        generate_synthetic(gk, v, deg, dim, seed, dsdir, dtype=dt)
        weights = random_weights(kind, dims, wseed, gin_epsilon=eps,
                                 gain=gain)
        REC.layers.clear()
        out = work / f"run_{case}"
        report = rt.run_inference(dsdir, weights, rt.PipelineConfig(**cfg),
                                  out)
        graph = read_csr(dsdir)
        feats = load_layer_matrix(dsdir / "features")
        rows = np.sort(np.random.default_rng(0).choice(v, SAMPLE_ROWS,
                                                       replace=False))
        entry = {"dataset": ds, "dataset_spec": SCALE_DATASETS[ds],
                 "model": int(kind), "dims": dims, "weight_seed": wseed,
                 "gin_epsilon": eps, "gain": gain, "config": cfg,
                 "num_edges": int(graph.num_edges), "layers": []}
        arrays = {"rows": rows}
        last = len(weights.layers) - 1
        for l, m in enumerate(report.layers):
            y = load_layer_matrix(out / f"layer_{l}")
            log = REC.layers[l]
            lay = {f: getattr(m, f) for f in METRIC_FIELDS}
            lay["output_sha"] = digest_array(y)
            lay["output_absmax"] = float(np.abs(y).max())
            for key in ("victims", "reloads", "graduated"):
                flat = flatten_events(log[key])
                lay[f"{key}_sha"] = digest_array(flat)
                lay[f"{key}_events"] = len(log[key])
            arrays[f"L{l}_out_rows"] = y[rows]
            trunc = ModelWeights(kind, weights.layers[:l + 1], eps)
            ref = oracle_inference(graph, feats, trunc, memory_cap=32 << 30)
            if l != last:
                np.maximum(ref, 0.0, out=ref)
            lay["oracle_absmax"] = float(np.abs(ref).max())
            arrays[f"L{l}_oracle_rows"] = ref[rows]
            del ref
            entry["layers"].append(lay)
            print(case, l, lay["messages"], lay["output_sha"][:12],
                  flush=True)
        entry["metrics_csv"] = metrics_rows(out / "metrics.csv")
        entry["layer_dirs"] = [dir_digest(out / f"layer_{l}")
                               for l in range(len(report.layers))]
        manifest[case] = entry
        np.savez_compressed(OUT / f"{case}.npz", **arrays)
        path.write_text(json.dumps(manifest, indent=1, sort_keys=True))


def reorder_goldens():
    """Greedy reordering (oocgnn/reorder.py): permutation, scores and the
    relabelled CSR of three graphs."""
    from oocgnn.reorder import build_order, relabel_graph, score_vertices
    work = Path(tempfile.mkdtemp(prefix="golden_reorder_"))
    out = {}
    for name in ("fig2", "uniform", "pa"):
        if name == "fig2":
            d = fig2_dataset(work)
        else:
            gk, v, deg, dim, seed, dt = DATASETS[name]
            d = work / name
            generate_synthetic(gk, v, deg, dim, seed, d, dtype=dt)
        g = read_csr(d)
        scores = score_vertices(g)
        o2n = build_order(g)
        rg = relabel_graph(g, o2n)
        out[name] = {"scores_sha": digest_array(scores),
                     "old_to_new_sha": digest_array(o2n),
                     "offsets_sha": digest_array(rg.offsets),
                     "neighbors_sha": digest_array(rg.neighbors),
                     "in_degrees_sha": digest_array(rg.in_degrees)}
        if name == "fig2":
            out[name]["old_to_new"] = o2n.tolist()
            out[name]["scores"] = scores.tolist()
    path = OUT / "golden.json"
    man = json.loads(path.read_text())
    man["_reorder"] = out
    path.write_text(json.dumps(man, indent=1, sort_keys=True))


if __name__ == "__main__":
    if sys.argv[1:] == ["reorder"]:
        reorder_goldens()
    elif sys.argv[1:] == ["scale"]:
        scale_goldens()
    else:
        main(set(sys.argv[1:]) or None)
