"""Chunk plan, chunk payloads and the layer-input loader.

* ``plan_chunks`` is the reference's chunk schedule, bit-exact
  (oocgnn/chunks.py:36-48): rows = max(1, budget // row_bytes).
* ``Chunk`` is the operator-path payload (oocgnn/chunks.py:204-220).
* ``load_layer_input`` replaces the merge-on-read spill reader
  (oocgnn/chunks.py:103-260) for the HBM-resident path: one sequential
  pass over the layer directory's spills into a pinned host buffer, ready
  for a single host->HBM copy. Every row is checked to arrive exactly once
  (the reference's delivery counters, criterion 2).
"""

from dataclasses import dataclass

import numpy as np

from .errors import ConsistencyError, CoverageError
from .storage import (
    NP_DTYPES,
    part_dir,
    read_layer_meta,
    read_manifest,
    read_spill_file,
)


def plan_chunks(num_vertices: int, dim: int, dtype: str, chunk_budget: int):
    row_bytes = dim * (2 if dtype == "f16" else 4)
    rows = max(1, chunk_budget // max(1, row_bytes))
    return [(s, min(s + rows, num_vertices))
            for s in range(0, num_vertices, rows)]


def chunk_rows(num_vertices: int, dim: int, dtype: str,
               chunk_budget: int) -> int:
    """Rows per chunk of plan_chunks (the plan is determined by it)."""
    row_bytes = dim * (2 if dtype == "f16" else 4)
    return max(1, chunk_budget // max(1, row_bytes))


@dataclass
class Chunk:
    start_id: int
    end_id: int
    features: np.ndarray       # (n, dim) f32 (or f16)
    local_offsets: np.ndarray  # (n+1,) int64, rebased to 0
    out_neighbors: np.ndarray  # int64 global destination ids

    @property
    def num_rows(self) -> int:
        return self.end_id - self.start_id


def chunk_from_csr(graph, features, start: int, end: int) -> Chunk:
    """Slice a chunk out of an in-memory CSR (the reference tests'
    ``chunk_of`` recipe, tests/test_orchestrator.py:61-70)."""
    o = graph.offsets
    lo, hi = int(o[start]), int(o[end])
    return Chunk(start, end, np.ascontiguousarray(features[start:end]),
                 (o[start:end + 1] - o[start]).astype(np.int64),
                 np.asarray(graph.neighbors[lo:hi], dtype=np.int64))


def load_layer_input(layer_dir, out=None):
    """Dense (V, dim) rows of a layer dir in their stored dtype.

    Returns (meta, rows, bytes_read, delivery) where delivery counts how
    often each id arrived (all ones, or CoverageError)."""
    meta = read_layer_meta(layer_dir)
    dtype = NP_DTYPES[meta.dtype]
    rows = out if out is not None else np.empty(
        (meta.num_vertices, meta.dim), dtype=dtype)
    delivery = np.zeros(meta.num_vertices, dtype=np.uint16)
    nbytes = 0
    for k in range(meta.partitions):
        pdir = part_dir(layer_dir, k)
        for name in read_manifest(pdir):
            ids, block = read_spill_file(pdir / name)
            if block.shape[1] != meta.dim or block.dtype != dtype:
                raise ConsistencyError(
                    f"{pdir / name}: shape {block.shape[1]}/{block.dtype} "
                    f"does not match layer meta {meta.dim}/{meta.dtype}")
            rows[ids] = block
            delivery[ids] += 1
            nbytes += block.nbytes + ids.nbytes
    if not np.all(delivery == 1):
        bad = np.flatnonzero(delivery != 1)
        raise CoverageError(
            f"{layer_dir}: {bad.size} ids not delivered exactly once, "
            f"first {bad[:8].tolist()}")
    return meta, rows, nbytes, delivery
