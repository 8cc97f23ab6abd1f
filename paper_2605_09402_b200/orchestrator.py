"""The per-layer operator triple on the GPU.

``init_layer`` / ``process_chunk`` / ``finalize_layer`` keep the signatures
and error behaviour of oocgnn/orchestrator.py:93-323 (the seam the
reference's own tests drive, tests/test_orchestrator.py:61-84). Each call
goes through the C-ABI (atlas_layer_create / atlas_chunk_submit /
atlas_chunk_graduated / atlas_layer_finish): the chunk is staged to HBM,
stable-sorted by destination, aggregated with the bit-exact f32 kernel,
and replayed through the exact control engine; graduated rows are handed
to ``sink.add_batch`` batch by batch in the reference's order.
"""

from dataclasses import dataclass, field

import numpy as np

from .engine import DeviceLayer, percentile99
from .errors import ConfigError, IncompleteLayerError
from .iostats import IOCounters, StageCounters
from .memstore import MemoryBudget, MemoryFacade, make_policy
from .storage import ModelKind, ModelWeights
from .vertexstate import StateTable


def make_message(h_source: np.ndarray, model: ModelKind,
                 in_degree_dest: int) -> np.ndarray:
    """Per-edge message (oocgnn/orchestrator.py:27-37), f32 semantics."""
    h = np.asarray(h_source, dtype=np.float32)
    if model in (ModelKind.GCN, ModelKind.SAGE):
        return h / np.float32(max(1, in_degree_dest))
    return h.copy()


@dataclass
class LayerMetrics:
    layer: int
    messages: int = 0
    evictions: int = 0
    reloads: int = 0
    unique_reloads: int = 0
    mean_span: float = 0.0
    p99_span: float = 0.0
    mean_reload_pct: float = 0.0
    bytes_read: int = 0
    bytes_written: int = 0
    wall_seconds: float = 0.0
    feature_bytes_read: int = 0
    hot_peak: int = 0
    hot_slot_count: int = 0
    delivery_counts: np.ndarray = field(default=None, repr=False)
    fast_path: bool = False
    gpu_seconds: float = 0.0
    agg_ms: float = 0.0
    control_ms: float = 0.0
    transform_ms: float = 0.0


CSV_FIELDS = [
    "layer", "messages", "evictions", "reloads", "unique_reloads",
    "mean_span", "p99_span", "mean_reload_pct", "bytes_read",
    "bytes_written", "wall_seconds",
]


@dataclass
class LayerContext:
    layer_index: int
    model: ModelKind
    num_vertices: int
    in_degrees: np.ndarray
    embed_dim: int
    agg_dim: int
    device_layer: DeviceLayer
    memory: MemoryFacade
    io: IOCounters
    counters: StageCounters
    gin_epsilon: float = 0.0
    self_term: bool = False
    mean_norm: bool = False
    sub_batch: int = 1
    chunks_seen: int = 0
    states: StateTable = None

    @property
    def pending(self) -> np.ndarray:
        return self.device_layer.state_arrays()[0]

    @property
    def first_step(self) -> np.ndarray:
        return self.device_layer.state_arrays()[2]

    @property
    def last_step(self) -> np.ndarray:
        return self.device_layer.state_arrays()[3]


def slot_budget(weights: ModelWeights, layer_index: int, hot_budget_bytes,
                hot_slots=None) -> MemoryBudget:
    agg = weights.agg_dim(layer_index)
    if hot_slots is not None:
        if hot_slots < 1:
            raise ConfigError("hot_slots must be >= 1")
        return MemoryBudget(hot_slots, agg)
    return MemoryBudget.from_bytes(hot_budget_bytes, agg)


def init_layer(in_degrees: np.ndarray, weights: ModelWeights,
               layer_index: int, *, hot_budget_bytes: int, cold_path=None,
               io: IOCounters = None, eviction: str = "minpend",
               seed: int = 0, hot_slots=None, evict_batch=None,
               dst_range=None, record_log: bool = False,
               device: int = 0) -> LayerContext:
    """oocgnn/orchestrator.py:93-145 on the device. ``cold_path`` is
    accepted for signature compatibility; evicted records stay in the
    device tier."""
    make_policy(eviction)
    budget = slot_budget(weights, layer_index, hot_budget_bytes, hot_slots)
    kind = weights.kind
    layer = DeviceLayer(
        in_degrees, int(kind), weights.embedding_dim(layer_index),
        weights.agg_dim(layer_index), budget.slot_count,
        gin_epsilon=weights.gin_epsilon, eviction=eviction, seed=seed,
        evict_batch=evict_batch, dst_range=dst_range, record_log=record_log,
        device=device)
    ctx = LayerContext(
        layer_index=layer_index, model=kind,
        num_vertices=len(in_degrees),
        in_degrees=np.asarray(in_degrees, dtype=np.int64),
        embed_dim=weights.embedding_dim(layer_index),
        agg_dim=weights.agg_dim(layer_index), device_layer=layer,
        memory=MemoryFacade(budget, evict_batch, layer),
        io=io if io is not None else IOCounters(),
        counters=StageCounters(), gin_epsilon=weights.gin_epsilon,
        self_term=kind in (ModelKind.SAGE, ModelKind.GIN),
        mean_norm=kind in (ModelKind.GCN, ModelKind.SAGE),
        sub_batch=max(1, budget.slot_count // 2))
    ctx.states = StateTable(lambda: layer.state_arrays()[1])
    return ctx


def process_chunk(ctx: LayerContext, chunk, sink) -> None:
    """oocgnn/orchestrator.py:216-299 for one chunk, on the GPU."""
    layer = ctx.device_layer
    layer.submit_chunk(chunk.start_id, chunk.end_id, chunk.features,
                       chunk.local_offsets, chunk.out_neighbors)
    ctx.chunks_seen += 1
    ids, rows, lens = layer.graduated(with_rows=True)
    pos = 0
    for n in lens.tolist():
        sink.add_batch(ids[pos:pos + n], rows[pos:pos + n])
        pos += n


def metrics_from_device(layer: DeviceLayer, layer_index: int) -> LayerMetrics:
    raw = layer.finish()
    m = LayerMetrics(layer=layer_index)
    m.messages = raw.messages
    m.evictions = raw.evictions
    m.reloads = raw.reloads
    m.unique_reloads = raw.unique_reloads
    if raw.span_count:
        m.mean_span = float(np.float64(raw.span_sum) / raw.span_count)
        m.p99_span = percentile99(raw.span_count, raw.span_q_lo,
                                  raw.span_q_hi)
    rel, tou = layer.chunk_stats()
    if len(rel):
        pcts = [100.0 * int(r) / max(1, int(t)) for r, t in zip(rel, tou)]
        m.mean_reload_pct = float(np.mean(pcts))
    m.hot_peak = raw.hot_peak
    m.hot_slot_count = raw.hot_slot_count
    m.fast_path = raw.fast_path
    m.bytes_read = raw.cold_bytes_read
    m.bytes_written = raw.cold_bytes_written
    return m


def finalize_layer(ctx: LayerContext) -> LayerMetrics:
    """oocgnn/orchestrator.py:302-323: completion check + metrics."""
    m = metrics_from_device(ctx.device_layer, ctx.layer_index)
    c = ctx.counters
    c.messages, c.evictions, c.reloads = m.messages, m.evictions, m.reloads
    c.hot_peak = m.hot_peak
    ctx.io.cold_bytes_read += m.bytes_read
    ctx.io.cold_bytes_written += m.bytes_written
    m.bytes_read = ctx.io.total_read()
    m.bytes_written = ctx.io.total_written()
    return m


__all__ = ["make_message", "LayerMetrics", "CSV_FIELDS", "LayerContext",
           "init_layer", "process_chunk", "finalize_layer",
           "IncompleteLayerError"]
