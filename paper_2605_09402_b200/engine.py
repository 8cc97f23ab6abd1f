"""Device-side objects behind the reference API: topology and layer state.

``DeviceGraph`` holds one destination range's CSR + CSC in HBM
(atlas_graph_create). ``DeviceLayer`` is the GPU LayerContext
(atlas_layer_create): pending counters, lifecycle states, the hot-slot
budget and its eviction policy, the f32 aggregation records, and the
integer logs. Both are thin owners of C-ABI handles; all compute happens in
libatlas_b200.so.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import ConfigError

DTYPE_CODES = {np.dtype(np.float32): N.F32, np.dtype(np.float16): N.F16}


def torch_dtype_code(t) -> int:
    import torch

    return {torch.float32: N.F32, torch.float16: N.F16,
            torch.bfloat16: N.BF16}[t.dtype]


def rnd_state_of(seed: int):
    """numpy default_rng(seed)'s PCG64 state as (hi, lo, inc_hi, inc_lo)."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    m = (1 << 64) - 1
    return (st["state"] >> 64, st["state"] & m, st["inc"] >> 64,
            st["inc"] & m)


class DeviceGraph:
    """CSR + destination-major view of [lo, hi) resident on one GPU."""

    def __init__(self, offsets, neighbors, in_degrees, dst_range=None,
                 device: int = 0, stream=None):
        lib = N.lib()
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        nbrs = np.ascontiguousarray(neighbors, dtype=np.uint32)
        self.in_degrees = np.ascontiguousarray(in_degrees, dtype=np.uint32)
        self.num_vertices = len(self.offsets) - 1
        self.num_edges = len(nbrs)
        lo, hi = dst_range if dst_range else (0, self.num_vertices)
        self.lo, self.hi = int(lo), int(hi)
        self.device = device
        h = ctypes.c_void_p()
        N.check(lib.atlas_graph_create(
            device, self.num_vertices, self.num_edges, N.ptr(self.offsets),
            N.ptr(nbrs), N.ptr(self.in_degrees), self.lo, self.hi,
            N.stream_handle(stream), ctypes.byref(h)))
        self.handle = h
        n = ctypes.c_int64()
        N.check(lib.atlas_graph_csc(h, None, None, ctypes.byref(n)))
        self.local_edges = n.value

    @classmethod
    def from_csr(cls, graph, **kw):
        return cls(graph.offsets, graph.neighbors, graph.in_degrees, **kw)

    def update(self, offsets, neighbors, in_degrees, stream=None):
        """Re-upload a CSR for the same destination range (host arrays:
        numpy, or pinned torch tensors for full-speed copies) and rebuild
        the CSC view in the existing device buffers."""
        def host(a, dtype):
            if isinstance(a, np.ndarray):
                return np.ascontiguousarray(a, dtype=dtype)
            return a
        off = host(offsets, np.int64)
        nb = host(neighbors, np.uint32)
        deg = host(in_degrees, np.uint32)
        v, e = len(off) - 1, len(nb)
        N.check(N.load_library().atlas_graph_update(
            self.handle, v, e, N.ptr(off), N.ptr(nb), N.ptr(deg),
            N.stream_handle(stream)))
        self.num_vertices, self.num_edges = v, e
        n = ctypes.c_int64()
        N.check(N.load_library().atlas_graph_csc(self.handle, None, None,
                                                 ctypes.byref(n)))
        self.local_edges = n.value
        self.version = getattr(self, "version", 0) + 1

    def close(self):
        if getattr(self, "handle", None):
            N.load_library().atlas_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class RawMetrics:
    messages: int
    evictions: int
    reloads: int
    unique_reloads: int
    admissions: int
    graduations: int
    hot_peak: int
    hot_slot_count: int
    chunks: int
    span_count: int
    span_sum: int
    span_q_lo: int
    span_q_hi: int
    cold_bytes_read: int
    cold_bytes_written: int
    fast_path: bool


class DeviceLayer:
    """One layer's engine state on the GPU (the LayerContext of
    oocgnn/orchestrator.py:68-145)."""

    def __init__(self, in_degrees, model: int, embed_dim: int, agg_dim: int,
                 slot_count: int, *, gin_epsilon: float = 0.0,
                 eviction: str = "minpend", seed: int = 0, evict_batch=None,
                 dst_range=None, record_log: bool = False,
                 force_exact: bool = False, device: int = 0, stream=None):
        lib = N.lib()
        if eviction not in N.POLICY_CODES:
            raise ConfigError(f"unknown eviction policy {eviction!r}")
        self.in_degrees = np.ascontiguousarray(in_degrees, dtype=np.uint32)
        v = len(self.in_degrees)
        lo, hi = dst_range if dst_range else (0, v)
        self.lo, self.hi = int(lo), int(hi)
        self.num_vertices = v
        self.model, self.embed_dim, self.agg_dim = model, embed_dim, agg_dim
        self.slot_count = int(slot_count)
        self.eviction = eviction
        self.record_log = record_log
        self.device = device
        d = N.LayerDesc()
        d.num_vertices = v
        d.dst_lo, d.dst_hi = self.lo, self.hi
        d.model = int(model)
        d.gin_epsilon = float(gin_epsilon)
        d.embed_dim, d.agg_dim = embed_dim, agg_dim
        d.slot_count = self.slot_count
        d.evict_batch = int(evict_batch or 0)
        d.policy = N.POLICY_CODES[eviction]
        d.record_log = int(record_log)
        if eviction == "rnd":
            for i, x in enumerate(rnd_state_of(seed)):
                d.rnd_state[i] = x
        d.device = device
        d.force_exact = int(force_exact)
        h = ctypes.c_void_p()
        N.check(lib.atlas_layer_create(ctypes.byref(d),
                                       N.ptr(self.in_degrees),
                                       N.stream_handle(stream),
                                       ctypes.byref(h)))
        self.handle = h
        self.h2d_bytes = 0

    def reset(self, stream=None):
        """init_layer again for a new pass, reusing device memory."""
        N.check(N.load_library().atlas_layer_reset(self.handle,
                                                   N.stream_handle(stream)))

    def bind_graph(self, graph: DeviceGraph, stream=None):
        """reset() after a topology refresh: in-degrees come from the
        graph's device copy."""
        N.check(N.load_library().atlas_layer_bind_graph(
            self.handle, graph.handle, N.stream_handle(stream)))

    # -- operator path ------------------------------------------------------
    def submit_chunk(self, start, end, rows, local_offsets, neighbors,
                     stream=None):
        rows = np.ascontiguousarray(rows)
        if rows.dtype not in DTYPE_CODES:
            rows = rows.astype(np.float32)
        off = np.ascontiguousarray(local_offsets, dtype=np.int64)
        nb = np.ascontiguousarray(neighbors, dtype=np.int64)
        n = end - start
        if rows.shape != (n, self.embed_dim):
            raise ConfigError(
                f"chunk rows {rows.shape} != ({n}, {self.embed_dim})")
        if off.shape != (n + 1,) or (n and (off[0] != 0 or off[-1] != len(nb))):
            raise ConfigError("chunk offsets do not bracket its neighbors")
        N.check(N.load_library().atlas_chunk_submit(
            self.handle, start, end, N.ptr(rows), DTYPE_CODES[rows.dtype],
            N.ptr(off), N.ptr(nb), len(nb), N.stream_handle(stream)))
        self.h2d_bytes += rows.nbytes + off.nbytes + nb.nbytes

    def graduated(self, with_rows=True):
        """(ids int64, rows f32 (n, agg_dim) or None, batch lengths)."""
        lib = N.load_library()
        cnt, nb = ctypes.c_int64(), ctypes.c_int64()
        N.check(lib.atlas_chunk_graduated(self.handle, None, None, 0,
                                          ctypes.byref(cnt), None, 0,
                                          ctypes.byref(nb)))
        ids = np.empty(cnt.value, dtype=np.int64)
        rows = (np.empty((cnt.value, self.agg_dim), dtype=np.float32)
                if with_rows else None)
        lens = np.empty(nb.value, dtype=np.int64)
        N.check(lib.atlas_chunk_graduated(
            self.handle, N.ptr(ids), N.ptr(rows), cnt.value,
            ctypes.byref(cnt), N.ptr(lens), nb.value, ctypes.byref(nb)))
        return ids, rows, lens

    # -- whole-layer path ---------------------------------------------------
    def run_resident(self, graph: DeviceGraph, x, chunk_rows: int,
                     input_flag=None, stream=None):
        """x: torch CUDA tensor (V, embed_dim) f32/f16/bf16. input_flag:
        the int32 CUDA tensor the transform that produced x filled (spares
        a scan of x), or None."""
        if x.shape[1] != self.embed_dim or x.shape[0] != self.num_vertices:
            raise ConfigError(f"input {tuple(x.shape)} does not match layer "
                              f"({self.num_vertices}, {self.embed_dim})")
        N.check(N.load_library().atlas_layer_run_resident(
            self.handle, graph.handle, x.data_ptr(), torch_dtype_code(x),
            x.stride(0), int(chunk_rows), N.ptr(input_flag),
            N.stream_handle(stream)))

    def run_blocked(self, graph: DeviceGraph, x, chunk_rows: int, weight,
                    bias, y, *, relu: bool, backend: int, block_rows: int,
                    input_flag=None, out_flag=None, stream=None):
        """Resident layer with bounded device records
        (atlas_layer_run_blocked): destinations aggregate and transform in
        blocks of ``block_rows`` records, the reference's graduated batches
        leaving the hot store (oocgnn/compute.py:125-205). Writes y."""
        if x.shape[1] != self.embed_dim or x.shape[0] != self.num_vertices:
            raise ConfigError(f"input {tuple(x.shape)} does not match layer "
                              f"({self.num_vertices}, {self.embed_dim})")
        N.check(N.load_library().atlas_layer_run_blocked(
            self.handle, graph.handle, x.data_ptr(), torch_dtype_code(x),
            x.stride(0), int(chunk_rows), N.ptr(input_flag), int(backend),
            weight.data_ptr(), bias.data_ptr(), weight.shape[0], int(relu),
            y.data_ptr(), torch_dtype_code(y), y.stride(0), N.ptr(out_flag),
            int(block_rows), N.stream_handle(stream)))

    def record_bytes(self) -> int:
        """Device bytes of f32 aggregation records the layer holds."""
        n = ctypes.c_int64()
        N.check(N.load_library().atlas_layer_record_bytes(
            self.handle, ctypes.byref(n)))
        return n.value

    def run_gat(self, graph: DeviceGraph, z, layout, bias, y, *,
                mean_heads: bool, relu: bool, chunk_rows: int,
                negative_slope: float = 0.2, attn_l=None, stream=None):
        """GAT pass B (atlas_layer_run_gat): z (V, ldz) CUDA tensor laid
        out as ``layout`` (gat.ZLayout) -> y (range rows) with bias, head
        concat/ReLU or head mean fused; control plane on the chunk plan.
        ``attn_l`` (f32 CUDA, heads x head_stride, zero pads) lets
        line-aligned f32 z (layout.line_rows) recompute el per edge."""
        if z.shape[0] != self.num_vertices or z.stride(1) != 1:
            raise ConfigError(f"z {tuple(z.shape)} does not cover the graph")
        N.check(N.load_library().atlas_layer_run_gat(
            self.handle, graph.handle, z.data_ptr(), torch_dtype_code(z),
            z.stride(0), layout.heads, layout.head_dim, layout.head_stride,
            layout.el_col, layout.er_col, bias.data_ptr(), int(mean_heads),
            int(relu),
            float(negative_slope), y.data_ptr(), torch_dtype_code(y),
            y.stride(0), N.ptr(attn_l), int(chunk_rows),
            N.stream_handle(stream)))

    def run_fused(self, graph: DeviceGraph, z, d: int, chunk_rows: int,
                  bias, y, *, data_model: int, relu: bool, self_rows=None,
                  input_flag=None, out_flag=None, host_out=None,
                  host_slices: int = 8, stream=None):
        """Transform-first pass (atlas_layer_run_fused): aggregate the first
        d columns of z (V x ldz f32, = h . W_z^T) with ``data_model``'s
        rule and write y = act(agg + self_rows + b) for the range
        (self_rows: SAGE's h_v . W2^T, one f32 row per local destination).
        ``host_out`` (pinned CPU tensor like y) also receives y, slice by
        slice, each D2H overlapping the next slice's aggregation."""
        if z.shape[0] != self.num_vertices or z.dtype.itemsize != 4:
            raise ConfigError(f"z {tuple(z.shape)} does not cover the graph")
        if self_rows is not None and (self_rows.shape[0] != self.hi - self.lo
                                      or self_rows.stride(1) != 1):
            raise ConfigError("self rows must cover the destination range")
        N.check(N.load_library().atlas_layer_run_fused(
            self.handle, graph.handle, z.data_ptr(), z.stride(0),
            int(data_model), int(d), int(chunk_rows), N.ptr(input_flag),
            bias.data_ptr(), N.ptr(self_rows),
            0 if self_rows is None else self_rows.stride(0), y.shape[1],
            int(relu),
            y.data_ptr(), torch_dtype_code(y), y.stride(0), N.ptr(out_flag),
            N.ptr(host_out), 0 if host_out is None else host_out.stride(0),
            int(host_slices), N.stream_handle(stream)))

    def run_streamed(self, graph: DeviceGraph, x_host, chunk_rows: int,
                     tile_bytes: int = 256 << 20, stream=None):
        """x_host: pinned CPU torch tensor (V, embed_dim); streamed to HBM
        in double-buffered tiles while earlier tiles aggregate."""
        if x_host.shape[1] != self.embed_dim or \
                x_host.shape[0] != self.num_vertices:
            raise ConfigError(f"input {tuple(x_host.shape)} does not match "
                              f"layer ({self.num_vertices}, {self.embed_dim})")
        row_bytes = x_host.stride(0) * x_host.element_size()
        tile_rows = max(1, tile_bytes // max(1, row_bytes))
        N.check(N.load_library().atlas_layer_run_streamed(
            self.handle, graph.handle, x_host.data_ptr(),
            torch_dtype_code(x_host), x_host.stride(0), int(tile_rows),
            int(chunk_rows), N.stream_handle(stream)))

    def run_pieces(self, graph: DeviceGraph, x, bounds, events,
                   chunk_rows: int, stream=None):
        """x: CUDA tensor (V, embed_dim) whose rows [bounds[t], bounds[t+1])
        land when torch.cuda.Event ``events[t]`` fires (None: already
        there); each piece is aggregated as soon as it lands
        (atlas_layer_run_pieces)."""
        if x.shape[1] != self.embed_dim or x.shape[0] != self.num_vertices:
            raise ConfigError(f"input {tuple(x.shape)} does not match "
                              f"layer ({self.num_vertices}, {self.embed_dim})")
        b = np.ascontiguousarray(bounds, dtype=np.int64)
        n = len(b) - 1
        handles = (ctypes.c_void_p * max(1, n))(
            *[(e.cuda_event if e is not None else None) for e in events])
        N.check(N.load_library().atlas_layer_run_pieces(
            self.handle, graph.handle, x.data_ptr(), torch_dtype_code(x),
            x.stride(0), b.ctypes.data, n, handles, int(chunk_rows),
            N.stream_handle(stream)))

    def accumulator_ptr(self):
        p, ld = ctypes.c_void_p(), ctypes.c_int64()
        N.check(N.load_library().atlas_layer_accumulator(
            self.handle, ctypes.byref(p), ctypes.byref(ld)))
        return p.value, ld.value

    def accumulator(self):
        """Host copy of the f32 aggregation records of [lo, hi)."""
        import torch

        p, ld = self.accumulator_ptr()
        n = self.hi - self.lo
        if not n:
            return torch.empty((0, ld), dtype=torch.float32, device="cuda")

        class _Records:  # zero-copy view of the library's device buffer
            __cuda_array_interface__ = {"shape": (n, ld), "typestr": "<f4",
                                        "data": (p, False), "version": 3}

        torch.cuda.current_stream().synchronize()
        return torch.as_tensor(_Records(), device="cuda").clone()

    # -- results ------------------------------------------------------------
    def finish(self) -> RawMetrics:
        m = N.LayerMetricsC()
        N.check(N.load_library().atlas_layer_finish(self.handle,
                                                    ctypes.byref(m)))
        if m.incomplete:
            N.raise_incomplete(m)
        return RawMetrics(
            m.messages, m.evictions, m.reloads, m.unique_reloads,
            m.admissions, m.graduations, m.hot_peak, m.hot_slot_count,
            m.chunks, m.span_count, m.span_sum, m.span_q_lo, m.span_q_hi,
            m.cold_bytes_read, m.cold_bytes_written, bool(m.fast_path))

    def timing(self):
        """(aggregate_ms, control_ms) of the last run_resident, measured
        with CUDA events on the launching stream."""
        ms = (ctypes.c_float * 2)()
        N.check(N.load_library().atlas_layer_timing(self.handle, ms, 2))
        return float(ms[0]), float(ms[1])

    def chunk_stats(self):
        lib = N.load_library()
        n = ctypes.c_int64()
        N.check(lib.atlas_layer_chunk_stats(self.handle, None, None, 0,
                                            ctypes.byref(n)))
        rel = np.empty(n.value, dtype=np.int64)
        tou = np.empty(n.value, dtype=np.int64)
        N.check(lib.atlas_layer_chunk_stats(self.handle, N.ptr(rel),
                                            N.ptr(tou), n.value,
                                            ctypes.byref(n)))
        return rel, tou

    def log(self, which: int) -> np.ndarray:
        lib = N.load_library()
        n = ctypes.c_int64()
        N.check(lib.atlas_layer_log(self.handle, which, None, 0,
                                    ctypes.byref(n)))
        out = np.empty(n.value, dtype=np.int64)
        N.check(lib.atlas_layer_log(self.handle, which, N.ptr(out), n.value,
                                    ctypes.byref(n)))
        return out

    def state_arrays(self):
        n = self.hi - self.lo
        pend = np.empty(n, dtype=np.uint32)
        st = np.empty(n, dtype=np.uint8)
        first = np.empty(n, dtype=np.int64)
        last = np.empty(n, dtype=np.int64)
        N.check(N.load_library().atlas_layer_state(
            self.handle, N.ptr(pend), N.ptr(st), N.ptr(first), N.ptr(last)))
        return pend, st, first, last

    def close(self):
        if getattr(self, "handle", None):
            N.load_library().atlas_layer_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def transform_device(x_ptr: int, rows: int, k: int, ldx: int, w, b,
                     relu: bool, y, backend_code: int, flag=None,
                     stream=None):
    """y = act(x . W^T + b) on the GPU; w, b, y torch CUDA tensors; flag
    (int32 CUDA tensor or None) receives the output extremes flag."""
    N.check(N.load_library().atlas_transform(
        backend_code, x_ptr, rows, k, ldx, w.data_ptr(), b.data_ptr(),
        w.shape[0], int(relu), y.data_ptr(), torch_dtype_code(y),
        y.stride(0), N.ptr(flag), N.stream_handle(stream)))


def transform_typed(x, w, b, relu: bool, y, backend_code: int, rows=None,
                    flag=None, stream=None):
    """y = act(x . W^T + b) with x a CUDA tensor of any engine dtype
    (f16/bf16 inputs need the tcgen05 backend)."""
    n = x.shape[0] if rows is None else rows
    N.check(N.load_library().atlas_transform_typed(
        backend_code, x.data_ptr(), torch_dtype_code(x), n, x.shape[1],
        x.stride(0), w.data_ptr(), b.data_ptr(), w.shape[0], int(relu),
        y.data_ptr(), torch_dtype_code(y), y.stride(0), N.ptr(flag),
        N.stream_handle(stream)))


def transform_er(x, w, b, y, n: int, er_w, er_col: int, heads: int,
                 head_stride: int, stream=None):
    """GAT pass A with er fused (atlas_transform_er): y[:, :n] = x . W^T + b
    and y[:, er_col + h] = z_h . a_r[h] (tcgen05 register-split kernels)."""
    N.check(N.load_library().atlas_transform_er(
        1, x.data_ptr(), torch_dtype_code(x), x.shape[0], x.shape[1],
        x.stride(0), w.data_ptr(), b.data_ptr(), n, y.data_ptr(),
        torch_dtype_code(y), y.stride(0), er_w.data_ptr(), er_col, heads,
        head_stride, N.stream_handle(stream)))


def percentile99(count: int, q_lo: int, q_hi: int) -> float:
    """np.percentile(spans, 99) from its two order statistics
    (numpy 'linear' method: virtual index (n-1)*0.99, _lerp)."""
    if count == 0:
        return 0.0
    vi = (count - 1) * (99 / 100)
    t = vi - np.floor(vi)
    a, b = float(q_lo), float(q_hi)
    diff = b - a
    if t >= 0.5:
        return float(b - diff * (1 - t))
    return float(a + diff * t)
