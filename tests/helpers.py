"""Shared test helpers: golden-case loading, digests, oracle drivers."""

import hashlib
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_2605_09402_b200 import storage as S

GOLDEN = Path(__file__).resolve().parent / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def digest_array(a) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(str(a.dtype).encode() + str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def flatten_events(events) -> np.ndarray:
    out = []
    for ev in events:
        out.append(len(ev))
        out.extend(int(x) for x in ev)
    return np.asarray(out, dtype=np.int64)


def unflatten(flat):
    flat = list(np.asarray(flat).tolist())
    out, i = [], 0
    while i < len(flat):
        n = flat[i]
        out.append(flat[i + 1:i + 1 + n])
        i += 1 + n
    return out


@lru_cache(maxsize=None)
def golden_manifest():
    return json.loads((GOLDEN / "golden.json").read_text())


def golden_arrays(case):
    return dict(np.load(GOLDEN / f"{case}.npz"))


def fig2_graph():
    edges = [(0, 1), (0, 3), (2, 3), (4, 1), (4, 3)]
    return S.edges_to_csr(np.array([e[0] for e in edges]),
                          np.array([e[1] for e in edges]), 6)


@lru_cache(maxsize=8)
def dataset(name):
    """(GraphCSR, features) of a golden dataset, rebuilt with the
    reference-identical generators."""
    if name == "fig2":
        feats = np.random.default_rng(3).uniform(-1, 1, (6, 8)).astype(
            np.float32)
        return fig2_graph(), feats
    kind, v, deg, dim, seed, dtype = golden_manifest()["_datasets"][name]
    return S.synthetic_in_memory(kind, v, deg, dim, seed, dtype)


def case_weights(entry):
    kind = S.ModelKind(entry["model"])
    return S.random_weights(kind, entry["dims"], entry["weight_seed"],
                            gin_epsilon=entry["gin_epsilon"],
                            gain=entry["gain"])


DEFAULT_CFG = dict(hot_budget=64 << 20, chunk_budget=8 << 20,
                   eviction="minpend", seed=0, hot_slots=None,
                   evict_batch=None)


def case_config(entry):
    cfg = dict(DEFAULT_CFG)
    cfg.update({k: v for k, v in entry["config"].items() if k in cfg})
    return cfg


def layer_plan(weights, layer, num_vertices, in_dtype, cfg):
    """(chunk_rows, slot_count) the reference uses for a layer."""
    dim = weights.embedding_dim(layer)
    item = 2 if in_dtype == "f16" else 4
    rows = max(1, cfg["chunk_budget"] // max(1, dim * item))
    agg = weights.agg_dim(layer)
    slots = cfg["hot_slots"] or cfg["hot_budget"] // (agg * 4)
    return rows, slots


def oracle_case(case):
    """Run the oracle engine over every layer of a golden case; returns
    list of (out f32, metrics, log)."""
    from oracle import engine as OE

    entry = golden_manifest()[case]
    graph, feats = dataset(entry["dataset"])
    weights = case_weights(entry)
    cfg = case_config(entry)
    in_dtype = "f16" if feats.dtype == np.float16 else "f32"
    h = feats
    res = []
    for l, lw in enumerate(weights.layers):
        rows, slots = layer_plan(weights, l, graph.num_vertices, in_dtype, cfg)
        out, m, log = OE.run_layer(
            graph.offsets, graph.neighbors, graph.in_degrees, h,
            int(weights.kind), lw.weight, lw.bias,
            relu=l != len(weights.layers) - 1,
            embed_dim=weights.embedding_dim(l), agg_dim=weights.agg_dim(l),
            chunk_rows=rows, slot_count=slots,
            gin_epsilon=weights.gin_epsilon, eviction=cfg["eviction"],
            seed=cfg["seed"], evict_batch=cfg["evict_batch"])
        res.append((out, m, log))
        h = out
        in_dtype = "f32"
    return res
