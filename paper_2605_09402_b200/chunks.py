"""Chunk plan, chunk payloads and the layer-input loader.

* ``plan_chunks`` is the reference's chunk schedule, bit-exact
  (oocgnn/chunks.py:36-48): rows = max(1, budget // row_bytes).
* ``Chunk`` is the operator-path payload (oocgnn/chunks.py:204-220).
* ``load_layer_input`` replaces the merge-on-read spill reader
  (oocgnn/chunks.py:103-260): the library reads the layer directory's
  spill files in parallel straight into a pinned host buffer, the source of
  the K1 host->HBM streamer. Every row is checked to arrive exactly once
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


def _pinned_rows(shape, dtype):
    """A page-locked host buffer for the K1 streamer when CUDA is usable,
    else plain memory (host-only use, e.g. format tools)."""
    try:
        import torch
        if torch.cuda.is_available():
            t = torch.empty(shape, dtype={np.dtype(np.float32): torch.float32,
                                          np.dtype(np.float16): torch.float16}
                            [np.dtype(dtype)], pin_memory=True)
            return t.numpy()
    except Exception:  # noqa: BLE001 - no torch / no device: plain memory
        pass
    return np.empty(shape, dtype=dtype)


def load_layer_input(layer_dir, out=None, threads: int = 0):
    """Dense (V, dim) rows of a layer dir in their stored dtype, read by
    the library's parallel spill reader (csrc/spillio.cu) straight into a
    pinned buffer (the source of the K1 host->HBM streamer); replaces the
    reference's merge-on-read SpillSet (oocgnn/chunks.py:103-260).

    Returns (meta, rows, bytes_read, delivery) where delivery counts how
    often each id arrived (all ones, or CoverageError)."""
    import ctypes

    from . import _native as N

    meta = read_layer_meta(layer_dir)
    dtype = NP_DTYPES[meta.dtype]
    rows = out if out is not None else _pinned_rows(
        (meta.num_vertices, meta.dim), dtype)
    if rows.shape != (meta.num_vertices, meta.dim) or rows.dtype != dtype \
            or not rows.flags.c_contiguous:
        raise ConsistencyError(f"{layer_dir}: output buffer does not match "
                               f"({meta.num_vertices}, {meta.dim}) "
                               f"{meta.dtype}")
    paths = [str(part_dir(layer_dir, k) / name)
             for k in range(meta.partitions)
             for name in read_manifest(part_dir(layer_dir, k))]
    arr = (ctypes.c_char_p * max(1, len(paths)))(
        *[p.encode() for p in paths])
    delivery = np.zeros(meta.num_vertices, dtype=np.uint16)
    nbytes = ctypes.c_int64()
    N.check(N.load_library().atlas_spill_read(
        arr, len(paths), N.F32 if meta.dtype == "f32" else N.F16, meta.dim,
        meta.num_vertices, rows.ctypes.data, delivery.ctypes.data,
        int(threads), ctypes.byref(nbytes)))
    return meta, rows, int(nbytes.value), delivery


def load_layer_device(layer_dir, threads: int = 0, device: int = 0):
    """Dense (V, dim) rows of a layer dir straight into a CUDA tensor
    (atlas_spill_read_device): each run of consecutive ids is one
    GPUDirect Storage read (storage -> HBM) when the cuFile driver is
    available, else a pinned-bounce stream on the copy engines -- the B200
    counterpart of the reference's direct-I/O reader (oocgnn/chunks.py:
    103-260, oocgnn/directio.py). Returns (meta, rows, bytes_read,
    delivery, used_gds)."""
    import ctypes

    import torch

    from . import _native as N

    meta = read_layer_meta(layer_dir)
    tdt = torch.float32 if meta.dtype == "f32" else torch.float16
    paths = [str(part_dir(layer_dir, k) / name)
             for k in range(meta.partitions)
             for name in read_manifest(part_dir(layer_dir, k))]
    arr = (ctypes.c_char_p * max(1, len(paths)))(
        *[p.encode() for p in paths])
    delivery = np.zeros(meta.num_vertices, dtype=np.uint16)
    nbytes = ctypes.c_int64()
    gds = ctypes.c_int32()
    lib = N.load_library()
    code = N.F32 if meta.dtype == "f32" else N.F16
    # damaged directories fail before any device memory is touched
    N.check(lib.atlas_spill_read_device(
        arr, len(paths), code, meta.dim, meta.num_vertices, None, None,
        int(threads), None, None))
    rows = torch.empty((meta.num_vertices, meta.dim), dtype=tdt,
                       device=f"cuda:{device}")
    torch.cuda.synchronize(device)  # rows is allocated before the reads
    N.check(lib.atlas_spill_read_device(
        arr, len(paths), code, meta.dim, meta.num_vertices, rows.data_ptr(),
        delivery.ctypes.data, int(threads), ctypes.byref(nbytes),
        ctypes.byref(gds)))
    return meta, rows, int(nbytes.value), delivery, bool(gds.value)


def write_layer_output(layer_dir, matrix: np.ndarray, partitions: int = 1,
                       dtype: str = "f32", threads: int = 0) -> int:
    """Write a (V, dim) output matrix as a partitioned layer directory with
    the library's parallel spill writer (csrc/spillio.cu): one spill per
    partition, the bytes storage.write_matrix_as_layer produces
    (oocgnn/storage.py:468-491, tested byte-for-byte). Returns the bytes
    written."""
    import ctypes

    from . import _native as N
    from .storage import LayerMeta, partition_ranges, write_layer_meta

    rows = np.ascontiguousarray(matrix, dtype=NP_DTYPES[dtype])
    v, dim = rows.shape
    write_layer_meta(layer_dir, LayerMeta(v, dim, dtype, partitions))
    lib = N.load_library()
    total = 0
    for k, (lo, hi) in enumerate(partition_ranges(v, partitions)):
        pdir = part_dir(layer_dir, k)
        pdir.mkdir(parents=True, exist_ok=True)
        nb = ctypes.c_int64()
        N.check(lib.atlas_spill_write(
            str(pdir).encode(), rows[lo:hi].ctypes.data if hi > lo else None,
            N.F32 if dtype == "f32" else N.F16, dim, dim, lo, hi,
            max(1, hi - lo), int(threads), ctypes.byref(nb)))
        total += int(nb.value)
    return total


def graduation_spills(grad_order, num_vertices: int, partitions: int,
                      dim: int, spill_buffer: int):
    """The reference writer's file layout for one layer output
    (oocgnn/writer.py:40-115): per partition, a buffer of
    ``max(1, spill_buffer // partitions // (dim*4 + 8))`` rows fills in
    graduation order and every full buffer (and the final partial one) is
    flushed as one spill sorted by id. Returns, per partition, (ids int64
    laid out spill after spill, spill_start int64[nspills+1])."""
    from .storage import partition_width

    order = np.asarray(grad_order, dtype=np.int64)
    if order.shape != (num_vertices,):
        raise ConsistencyError(f"graduation order holds {order.size} ids, "
                               f"expected {num_vertices}")
    width = partition_width(num_vertices, partitions)
    per = max(1, spill_buffer // max(1, partitions) // (dim * 4 + 8))
    part = order // width
    out = []
    for k in range(partitions):
        seq = order[part == k]            # graduation order within k
        spill = np.arange(seq.size, dtype=np.int64) // per
        ids = seq[np.lexsort((seq, spill))]
        nsp = -(-seq.size // per)
        start = np.minimum(np.arange(nsp + 1, dtype=np.int64) * per,
                           seq.size)
        out.append((ids, start))
    return out


def write_graduation_layout(layer_dir, matrix: np.ndarray, grad_order,
                            partitions: int, spill_buffer: int,
                            threads: int = 0) -> int:
    """Write a (V, dim) layer output exactly as the reference's writer
    stage would have (same spill files, bytes and manifests, f32 rows --
    oocgnn/writer.py:60-62), given the layer's graduation order. Returns
    the spill bytes written (IOCounters.spill_bytes_written)."""
    import ctypes

    from . import _native as N
    from .storage import LayerMeta, write_layer_meta

    rows = np.ascontiguousarray(matrix, dtype=np.float32)
    v, dim = rows.shape
    layout = graduation_spills(grad_order, v, partitions, dim, spill_buffer)
    write_layer_meta(layer_dir, LayerMeta(v, dim, "f32", partitions))
    lib = N.load_library()
    total = 0
    for k, (ids, start) in enumerate(layout):
        pdir = part_dir(layer_dir, k)
        pdir.mkdir(parents=True, exist_ok=True)
        nb = ctypes.c_int64()
        N.check(lib.atlas_spill_write_runs(
            str(pdir).encode(), rows.ctypes.data, N.F32, dim, dim,
            ids.ctypes.data, start.ctypes.data, len(start) - 1,
            int(threads), ctypes.byref(nb)))
        total += int(nb.value)
    return total
