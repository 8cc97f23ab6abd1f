"""Greedy vertex reordering (oocgnn/reorder.py), computed on the GPU.

``score_vertices`` / ``build_order`` / ``relabel_graph`` keep the
reference's names and results bit-for-bit (float64 scores folded per source
in CSR order, stable descending sort with ties by ascending old id, rows
re-sorted ascending); the work runs in csrc/reorder.cu through
``atlas_reorder``. ``reorder_dataset`` writes the relabelled topology,
``perm.bin`` and the relabelled features in the reference's formats.
``compute_span`` is the reference's offline span replay (GCN stream
positions), kept for the reordering experiments.
"""

from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native as N
from .chunks import load_layer_input
from .errors import ConfigError
from .storage import (GraphCSR, read_csr, write_csr, write_matrix_as_layer,
                      write_permutation)


def _device_reorder(graph: GraphCSR):
    lib = N.lib()
    v, e = graph.num_vertices, graph.num_edges
    off = np.ascontiguousarray(graph.offsets, dtype=np.int64)
    nb = np.ascontiguousarray(graph.neighbors, dtype=np.uint32)
    deg = np.ascontiguousarray(graph.in_degrees, dtype=np.uint32)
    o2n = np.empty(v, dtype=np.int64)
    noff = np.empty(v + 1, dtype=np.int64)
    nnb = np.empty(e, dtype=np.uint32)
    ndeg = np.empty(v, dtype=np.uint32)
    scores = np.empty(v, dtype=np.float64)
    N.check(lib.atlas_reorder(0, v, e, N.ptr(off), N.ptr(nb), N.ptr(deg),
                              N.ptr(o2n), N.ptr(noff), N.ptr(nnb),
                              N.ptr(ndeg), N.ptr(scores),
                              N.stream_handle()))
    relabelled = GraphCSR(v, e, noff, nnb.astype(np.int64),
                          ndeg.astype(np.int64))
    return scores, o2n, relabelled


def score_vertices(graph: GraphCSR) -> np.ndarray:
    """oocgnn/reorder.py:30-44."""
    return _device_reorder(graph)[0]


def build_order(graph: GraphCSR) -> np.ndarray:
    """old_to_new (oocgnn/reorder.py:47-54)."""
    return _device_reorder(graph)[1]


def random_order(num_vertices: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).permutation(num_vertices).astype(
        np.int64)


def relabel_graph(graph: GraphCSR, old_to_new: np.ndarray) -> GraphCSR:
    """Apply a permutation (oocgnn/reorder.py:62-88). The greedy order's
    relabelling comes straight from the device pass; other permutations
    are applied with the same row-gather + per-row sort on the host."""
    v = graph.num_vertices
    if len(old_to_new) != v:
        raise ConfigError("permutation length != |V|")
    new_to_old = np.empty(v, dtype=np.int64)
    new_to_old[old_to_new] = np.arange(v, dtype=np.int64)
    new_out = np.diff(graph.offsets)[new_to_old]
    offsets = np.zeros(v + 1, dtype=np.int64)
    np.cumsum(new_out, out=offsets[1:])
    starts = graph.offsets[new_to_old]
    within = np.arange(graph.num_edges) - np.repeat(offsets[:-1], new_out)
    nbrs = np.asarray(old_to_new)[graph.neighbors[
        np.repeat(starts, new_out) + within]]
    rows = np.repeat(np.arange(v), new_out)
    nbrs = nbrs[np.lexsort((nbrs, rows))]
    return GraphCSR(v, graph.num_edges, offsets, nbrs,
                    graph.in_degrees[new_to_old])


def reorder_dataset(graph_dir, out_dir, *, ordering: str = "greedy",
                    partitions: int = 1, seed: int = 0) -> np.ndarray:
    """oocgnn/reorder.py:134-158."""
    graph_dir, out_dir = Path(graph_dir), Path(out_dir)
    graph = read_csr(graph_dir)
    if ordering == "greedy":
        _, old_to_new, relabelled = _device_reorder(graph)
    elif ordering in ("random", "original"):
        old_to_new = (random_order(graph.num_vertices, seed)
                      if ordering == "random"
                      else np.arange(graph.num_vertices, dtype=np.int64))
        relabelled = relabel_graph(graph, old_to_new)
    else:
        raise ConfigError(f"unknown ordering {ordering!r}")
    out_dir.mkdir(parents=True, exist_ok=True)
    write_csr(relabelled, out_dir)
    write_permutation(out_dir / "perm.bin", old_to_new)
    if (graph_dir / "features").exists():
        meta, rows, _, _ = load_layer_input(graph_dir / "features")
        moved = np.empty_like(rows, dtype=np.float32)
        moved[old_to_new] = rows
        write_matrix_as_layer(out_dir / "features", moved,
                              partitions=partitions)
    return old_to_new


@dataclass
class SpanStats:
    mean_span: float
    p99_span: float
    max_span: float


def compute_span(graph: GraphCSR) -> SpanStats:
    """Per-destination message spans of the source-order walk
    (oocgnn/reorder.py:168-187, an offline analysis helper).

    Message t of the walk is CSR edge t, so a destination's first and last
    steps are the smallest and largest CSR positions holding its id: a
    stable sort of the neighbour array groups each destination's positions
    in ascending order, and the run ends give both. Spans come out in
    ascending destination order, as the reference's masked arrays do."""
    nbrs = np.asarray(graph.neighbors)
    if nbrs.size == 0:
        return SpanStats(0.0, 0.0, 0.0)
    pos = np.argsort(nbrs, kind="stable")
    grouped = nbrs[pos]
    heads = np.flatnonzero(np.r_[True, grouped[1:] != grouped[:-1]])
    tails = np.r_[heads[1:], grouped.size] - 1
    spans = (pos[tails] - pos[heads]).astype(np.float64)
    return SpanStats(float(spans.mean()), float(np.percentile(spans, 99)),
                     float(spans.max()))
