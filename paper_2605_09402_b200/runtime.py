"""Public layer-wise inference API on the B200 engine.

Same entry points as oocgnn/runtime.py:60-329 — ``PipelineConfig``,
``run_layer``, ``run_inference``, ``write_metrics_csv``,
``final_layer_dir``, ``compare_outputs``, ``clone_config`` — reading and
writing the reference's dataset / layer-directory / weights formats.

What changes underneath: the reference's four Python
threads (reader -> orchestrator -> compute -> writer) become
  host loader -> one H2D copy of the layer input into HBM
  -> ``atlas_layer_run_resident`` (bit-exact scatter-aggregate over the
     destination-major view + the pending/eviction control plane on the
     reference chunk plan)
  -> ``atlas_transform`` (stable SIMT or tcgen05 backend)
  -> next layer's embeddings stay in HBM; the layer directory is written
     from one D2H copy.
``Engine`` is the device-resident core used by ``run_inference`` and by
bench.py; it also runs one destination range per GPU rank, exchanging the
layer outputs with an NCCL all-gather between layers.
"""

from __future__ import annotations

import csv
import shutil
import time
from dataclasses import dataclass, field, replace
from pathlib import Path

import numpy as np

from .chunks import chunk_rows as plan_rows
from .chunks import load_layer_input, write_layer_output
from .compute import device_code, get_backend
from .engine import DeviceGraph, DeviceLayer, transform_device
from .errors import ConfigError
from .exchange import gather_ranges
from .iostats import IOCounters
from .orchestrator import CSV_FIELDS, LayerMetrics, metrics_from_device
from .orchestrator import slot_budget
from .storage import (
    INDEGREE_FILE,
    TOPOLOGY_FILE,
    ModelKind,
    ModelWeights,
    load_layer_matrix,
    partition_ranges,
    read_in_degrees,
    read_layer_meta,
    read_topology_arrays,
    read_weights,
    write_matrix_as_layer,
)


@dataclass
class PipelineConfig:
    """oocgnn/runtime.py:60-85 plus the device knobs (last block)."""

    hot_budget: int = 64 << 20
    chunk_budget: int = 8 << 20
    graduation_budget: int = 16 << 20
    spill_buffer: int = 8 << 20
    partitions: int = 8
    queue_capacity: int = 20
    eviction: str = "minpend"
    seed: int = 0
    direct_io: bool = True
    discard_intermediate: bool = False
    hot_slots: int | None = None
    evict_batch: int | None = None
    max_open_files: int = 128
    backend: object = field(default=None, repr=False)
    # device knobs
    device: int = 0
    embed_dtype: str = "f32"       # next-layer embedding store: f32|f16|bf16
    record_log: bool = False        # keep victim/reload/graduation logs
    force_exact: bool = False       # always replay the exact control engine
    stream_tile_bytes: int = 256 << 20  # host->HBM tile of a streamed input
    # tcgen05 backend: when a layer's output is narrower than what it
    # aggregates, transform first and aggregate z = h . W^T (linearity of
    # the mean / sum); the bit-exact "stable" backend never does
    transform_first: bool = True
    # multi-GPU exchange: each owner range is broadcast in up to this many
    # pieces, and the next layer folds every piece in as it lands
    exchange_pieces: int = 4
    # bound the device records by the hot budget: destinations aggregate
    # and transform in blocks of the layer's slot count, so the f32 records
    # of at most that many vertices are ever resident (the reference's
    # graduated batches leaving the hot store); same bits as the unbounded
    # pass. Device backends and resident inputs only.
    bound_records: bool = False

    def validate(self) -> None:
        if self.partitions < 1:
            raise ConfigError("partitions must be >= 1")
        if self.queue_capacity < 1:
            raise ConfigError("queue capacity must be >= 1")
        if self.chunk_budget < 1:
            raise ConfigError("chunk budget must be positive")
        if self.embed_dtype not in ("f32", "f16", "bf16"):
            raise ConfigError(f"unknown embed dtype {self.embed_dtype!r}")


@dataclass
class RunReport:
    layers: list
    out_dir: Path
    wall_seconds: float

    def total(self, field_name: str):
        return sum(getattr(m, field_name) for m in self.layers)


def write_metrics_csv(path, layers) -> None:
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(CSV_FIELDS)
        for m in layers:
            w.writerow([m.layer, m.messages, m.evictions, m.reloads,
                        m.unique_reloads, f"{m.mean_span:.3f}",
                        f"{m.p99_span:.3f}", f"{m.mean_reload_pct:.3f}",
                        m.bytes_read, m.bytes_written,
                        f"{m.wall_seconds:.3f}"])


def _torch_dtype(name):
    import torch

    return {"f32": torch.float32, "f16": torch.float16,
            "bf16": torch.bfloat16}[name]


def _plan_dtype(layer_index: int, x) -> str:
    """Row format the reference's chunk plan sizes layer ``layer_index`` by
    (oocgnn/chunks.py:36-48 over the layer directory it reads): the dataset
    dtype for layer 0, f32 for every later layer because the reference's
    writer always emits f32 (oocgnn/writer.py:60-62) -- whatever dtype this
    engine keeps the embeddings in (``embed_dtype``)."""
    import torch

    if layer_index > 0:
        return "f32"
    return "f32" if x.dtype == torch.float32 else "f16"


class Engine:
    """Device-resident layer-wise inference over one destination range.

    graph: storage.GraphCSR; weights: ModelWeights. With ``dist`` (a
    torch.distributed group of G ranks) rank g owns
    partition_ranges(V, G)[g] and the layer outputs are all-gathered
    (NCCL) so every rank holds the next layer's full input."""

    def __init__(self, graph, weights: ModelWeights, config: PipelineConfig,
                 *, rank: int = 0, world: int = 1, dist_group=None):
        import torch

        config.validate()
        self.config = config
        self.weights = weights
        self.kind = weights.kind
        self.rank, self.world, self.group = rank, world, dist_group
        self.num_vertices = graph.num_vertices
        self.in_degrees = np.asarray(graph.in_degrees, dtype=np.uint32)
        self.ranges = partition_ranges(graph.num_vertices, world)
        self.lo, self.hi = self.ranges[rank]
        self.device = config.device
        torch.cuda.set_device(self.device)
        self.graph = DeviceGraph(graph.offsets, graph.neighbors,
                                 graph.in_degrees, (self.lo, self.hi),
                                 device=self.device)
        self.backend = get_backend(config.backend)
        self.W = [torch.as_tensor(np.ascontiguousarray(lw.weight)).cuda()
                  for lw in weights.layers]
        self.b = [torch.as_tensor(np.ascontiguousarray(lw.bias)).cuda()
                  for lw in weights.layers]
        self.exchange = None
        if world > 1:
            from .exchange import RangeExchange
            self.exchange = RangeExchange(graph.num_vertices, self.ranges,
                                          rank, dist_group,
                                          config.exchange_pieces)
        self._wz = {}
        self.last_layers = []
        self._layers = {}
        self.out_flags = {}
        self.z_flags = {}

    def close(self):
        for layer in self._layers.values():
            layer.close()
        self._layers.clear()
        self.graph.close()

    def transform_first(self, l: int) -> bool:
        """Whether layer l aggregates z = h . W_z^T instead of h: tcgen05
        backend only, and only when that narrows the aggregated width (the
        fused ring pass takes up to 128 f32 columns)."""
        if not self.config.transform_first or \
                device_code(self.backend) != 1:
            return False
        d = self.weights.embedding_dim(l)
        npad = -(-self.weights.layers[l].out_dim // 4) * 4
        return npad < d and npad <= 128 and d % 4 == 0

    def _z_weight(self, l: int):
        """(W_z, zero bias, padded width): W_z = W (GCN/GIN) or [W1; W2]
        (SAGE's mean half and self half), each padded to a multiple of 4
        rows so z rows are 16-byte aligned."""
        import torch

        if l in self._wz:
            return self._wz[l]
        lw = self.weights.layers[l]
        d = self.weights.embedding_dim(l)
        n = lw.out_dim
        npad = -(-n // 4) * 4
        parts = ([lw.weight[:, :d], lw.weight[:, d:]]
                 if self.kind == ModelKind.SAGE else [lw.weight])
        wz = np.zeros((npad * len(parts), d), dtype=np.float32)
        for i, p in enumerate(parts):
            wz[i * npad:i * npad + n] = p
        out = (torch.as_tensor(wz).cuda(),
               torch.zeros(wz.shape[0], device="cuda"), npad)
        self._wz[l] = out
        return out

    def layer(self, l: int, x, *, chunk_budget=None, input_flag=None,
              defer_metrics: bool = False, host_out=None, out=None,
              pieces=None):
        """One layer: x (V, d) CUDA tensor (or pinned host tensor, streamed)
        -> (y (V or range, out), metrics, device layer handle).
        ``input_flag``: extremes flag of the transform that produced x; the
        output's flag is left in ``self.out_flags[l]``. ``out``: where to
        write the (nloc, out) output (a rank's slice of the next layer's
        exchange buffer). ``pieces``: (bounds, events) of an input that is
        still arriving from the other ranks (RangeExchange.start).
        With ``defer_metrics`` nothing waits for the device: the second
        element is a callable that collects the metrics later (the layer's
        control-plane verdict and timings are taken then)."""
        import torch

        cfg = self.config
        w = self.weights
        last = l == len(w.layers) - 1
        t0 = time.perf_counter()
        d = w.embedding_dim(l)
        if x.shape[1] != d:
            raise ConfigError(
                f"layer {l} expects {d}-wide rows, input holds {x.shape[1]}")
        rows = plan_rows(self.num_vertices, d, _plan_dtype(l, x),
                         chunk_budget or cfg.chunk_budget)
        layer = self._layers.get(l)
        gv = getattr(self.graph, "version", 0)
        if layer is not None and layer.handle:
            # same descriptor: reuse the device workspaces
            if layer.graph_version == gv:
                layer.reset()
        else:
            budget = slot_budget(w, l, cfg.hot_budget, cfg.hot_slots)
            layer = DeviceLayer(
                self.in_degrees, int(self.kind), d, w.agg_dim(l),
                budget.slot_count, gin_epsilon=w.gin_epsilon,
                eviction=cfg.eviction, seed=cfg.seed,
                evict_batch=cfg.evict_batch, dst_range=(self.lo, self.hi),
                record_log=cfg.record_log, force_exact=cfg.force_exact,
                device=self.device)
            self._layers[l] = layer
            layer.graph_version = 0  # built from the initial host degrees
        if layer.graph_version != gv:
            # topology refreshed since: in-degrees from the device graph
            layer.bind_graph(self.graph)
            layer.graph_version = gv
        nloc = self.hi - self.lo
        out_dim = w.layers[l].out_dim
        y = out if out is not None else torch.empty(
            (nloc, out_dim), dtype=_torch_dtype(cfg.embed_dtype),
            device="cuda")
        if self.transform_first(l):
            return self._layer_transform_first(l, x, layer, rows, y, last,
                                               t0, defer_metrics, host_out)
        code = device_code(self.backend)
        if cfg.bound_records and x.is_cuda and pieces is None and \
                code is not None:
            return self._layer_blocked(l, x, layer, rows, y, last, t0,
                                       defer_metrics, host_out, input_flag,
                                       code)
        if not x.is_cuda and self.world > 1 and x.shape[0] == nloc \
                and nloc != self.num_vertices:
            # a rank holding only its own rows (its partition of the layer
            # input): upload them and all-gather the full input (SURVEY.md
            # §8e: every source row reaches every rank once per layer)
            x = self.gather(x.to("cuda", non_blocking=True))
        if x.is_cuda and pieces is not None:
            layer.run_pieces(self.graph, x, pieces[0], pieces[1], rows)
        elif x.is_cuda:
            layer.run_resident(self.graph, x, rows, input_flag=input_flag)
        else:  # host (pinned) input: stream it in tiles (K1 streamer)
            layer.run_streamed(self.graph, x, rows,
                               tile_bytes=self.config.stream_tile_bytes)
        acc_ptr, ld = layer.accumulator_ptr()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        if nloc:
            if code is not None:
                if l not in self.out_flags:
                    self.out_flags[l] = torch.zeros(1, dtype=torch.int32,
                                                    device="cuda")
                transform_device(acc_ptr, nloc, w.agg_dim(l), ld, self.W[l],
                                 self.b[l], not last, y, code,
                                 flag=self.out_flags[l])
            else:  # host plug-in backend (reference MatmulBackend protocol)
                from .compute import transform
                agg = layer.accumulator()[:, :w.agg_dim(l)].cpu().numpy()
                y.copy_(torch.as_tensor(transform(
                    agg, w.layers[l], apply_activation=not last,
                    backend=self.backend)))
        ev1.record()
        if host_out is not None:
            host_out.copy_(y, non_blocking=True)

        def collect():
            m = metrics_from_device(layer, l)
            m.agg_ms, m.control_ms = layer.timing()
            m.transform_ms = ev0.elapsed_time(ev1)
            m.gpu_seconds = time.perf_counter() - t0
            return m

        if defer_metrics:
            return y, collect, layer
        return y, collect(), layer

    def _layer_blocked(self, l, x, layer, rows, y, last, t0, defer_metrics,
                       host_out, input_flag, code):
        """Aggregate + transform in blocks of the slot budget: device
        records never exceed slot_count x agg_dim f32."""
        import torch

        if l not in self.out_flags:
            self.out_flags[l] = torch.zeros(1, dtype=torch.int32,
                                            device="cuda")
        layer.run_blocked(self.graph, x, rows, self.W[l], self.b[l], y,
                          relu=not last, backend=code,
                          block_rows=layer.slot_count, input_flag=input_flag,
                          out_flag=self.out_flags[l])
        if host_out is not None:
            host_out.copy_(y, non_blocking=True)

        def collect():
            m = metrics_from_device(layer, l)
            m.agg_ms, m.control_ms = layer.timing()
            m.transform_ms = 0.0  # inside agg_ms, block by block
            m.gpu_seconds = time.perf_counter() - t0
            return m

        if defer_metrics:
            return y, collect, layer
        return y, collect(), layer

    def _transform_rows(self, l, x, wz, zb, out=None):
        """z = x . W_z^T (f32) on tcgen05; a pinned host x streams to HBM
        in double-buffered row tiles on a side stream, each tile
        transformed as soon as it lands (layer-input ingest overlaps the
        GEMM). Leaves z's extremes flag in self.z_flags[l]."""
        import torch

        from .engine import transform_typed

        if l not in self.z_flags:
            self.z_flags[l] = torch.zeros(1, dtype=torch.int32, device="cuda")
        n = x.shape[0]
        # row pitch: whole 64-byte units, so a narrow z row never straddles
        # more DRAM bursts than it needs (the GEMM writes wz.shape[0] cols)
        z = out if out is not None else torch.empty(
            (n, z_pitch(wz.shape[0])), dtype=torch.float32, device="cuda")
        if x.is_cuda:
            if n:
                transform_typed(x, wz, zb, False, z, 1, flag=self.z_flags[l])
            else:
                self.z_flags[l].zero_()
            return z
        row_b = x.stride(0) * x.element_size()
        tile = max(128, (self.config.stream_tile_bytes // row_b) // 128 * 128)
        ntiles = -(-n // tile)
        if getattr(self, "_copy_stream", None) is None:
            self._copy_stream = torch.cuda.Stream()
        copy, cur = self._copy_stream, torch.cuda.current_stream()
        bufs = [torch.empty((min(tile, n), x.shape[1]), dtype=x.dtype,
                            device="cuda") for _ in range(min(2, ntiles))]
        flags = torch.zeros(max(1, ntiles), dtype=torch.int32, device="cuda")
        freed = [None, None]
        for t in range(ntiles):
            b, r0 = t & 1, t * tile
            r1 = min(n, r0 + tile)
            with torch.cuda.stream(copy):
                if freed[b] is not None:
                    copy.wait_event(freed[b])
                bufs[b][:r1 - r0].copy_(x[r0:r1], non_blocking=True)
                ready = torch.cuda.Event()
                ready.record(copy)
            cur.wait_event(ready)
            transform_typed(bufs[b][:r1 - r0], wz, zb, False, z[r0:r1], 1,
                            flag=flags[t:t + 1])
            freed[b] = torch.cuda.Event()
            freed[b].record(cur)
        torch.amax(flags, dim=0, keepdim=True, out=self.z_flags[l])
        return z

    def _layer_transform_first(self, l, x, layer, rows, y, last, t0,
                               defer_metrics, host_out=None):
        """z = h . W_z^T on tcgen05 for every source row, then one fused
        pass: control plane on the reference chunk plan + ring aggregation
        of z + bias / SAGE self half / ReLU epilogue (no f32 records)."""
        import torch

        from .engine import transform_typed

        wz, zb, npad = self._z_weight(l)
        # with G ranks each rank transforms its own rows and the z rows are
        # all-gathered (z is narrower than h, so this is the cheap exchange)
        if self.world > 1 and x.shape[0] == self.num_vertices:
            x = x[self.lo:self.hi]
        sage = self.kind == ModelKind.SAGE
        ex = self.exchange
        zfull = None
        if ex is not None and not sage:
            # the GEMM writes this rank's z rows straight into its slice of
            # the exchange buffer; the owners' broadcasts fill the rest
            zfull = ex.buffer(("z", l), z_pitch(wz.shape[0]), torch.float32,
                              "cuda")
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        zp = self._transform_rows(
            l, x, wz, zb, out=None if zfull is None else ex.own(zfull))
        ev[1].record()
        # SAGE's self half z2 = h_v . W2^T is needed for local rows only
        self_rows = None
        if sage:
            self_rows = zp[:, npad:] if self.world > 1 else \
                zp[self.lo:self.hi, npad:]
        z = zp
        if ex is not None:
            if sage:  # exchange z1 only, in its own 64-byte-pitch rows
                zfull = ex.buffer(("z1", l), z_pitch(npad), torch.float32,
                                  "cuda")
                ex.own(zfull)[:, :npad].copy_(zp[:, :npad])
            _, events = ex.start(zfull)
            ex.finish(events)
            z = zfull
        elif self.world > 1:  # a subclass's own gather (bench rank slice)
            if sage:
                z1 = torch.zeros((zp.shape[0], z_pitch(npad)),
                                 dtype=zp.dtype, device="cuda")
                z1[:, :npad] = zp[:, :npad]
                zp = z1
            z = self.gather(zp)
        if self.world > 1:
            self.allreduce_max(self.z_flags[l])
        if l not in self.out_flags:
            self.out_flags[l] = torch.zeros(1, dtype=torch.int32,
                                            device="cuda")
        data_model = (ModelKind.GIN if self.kind == ModelKind.GIN
                      else ModelKind.GCN)
        layer.run_fused(self.graph, z, npad, rows, self.b[l], y,
                        data_model=int(data_model), relu=not last,
                        self_rows=self_rows,
                        input_flag=self.z_flags[l],
                        out_flag=self.out_flags[l], host_out=host_out)

        def collect():
            m = metrics_from_device(layer, l)
            m.agg_ms, m.control_ms = layer.timing()
            m.transform_ms = ev[0].elapsed_time(ev[1])
            m.gpu_seconds = time.perf_counter() - t0
            return m

        if defer_metrics:
            return y, collect, layer
        return y, collect(), layer

    def update_graph(self, offsets, neighbors, in_degrees):
        """Refresh the topology (same vertex count and range) without
        reallocating; cached layers re-read their in-degrees from the
        device graph on their next pass (atlas_layer_bind_graph)."""
        self.graph.update(offsets, neighbors, in_degrees)

    def allreduce_max(self, t):
        """Element-wise max over ranks (the extremes flags)."""
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)

    def gather(self, y_local):
        """All ranks' ranges -> full (V, out) tensor, by owner broadcasts
        into one buffer (exchange.RangeExchange; NCCL on GPUs)."""
        if self.world == 1:
            return y_local
        return self.exchange.gather(y_local, key=("in", y_local.shape[1],
                                                  y_local.dtype))

    def infer(self, x, keep_layers: bool = False, host_out=None,
              metrics: bool = True):
        """All layers; returns (final local output, [LayerMetrics]).
        ``host_out`` (pinned CPU tensor of the output's shape and dtype)
        receives the final output too; a transform-first last layer copies
        it out slice by slice while it is still being computed. With
        ``metrics=False`` nothing waits for the device (metrics None): the
        control plane's verdicts are still taken when the layers are
        re-armed, but their counters are not read back."""
        import torch

        pending, outs = [], []
        h, flag, pieces = x, None, None
        nl = len(self.weights.layers)
        ex = self.exchange
        for l in range(nl):
            # with G ranks an aggregate-first next layer reads every rank's
            # rows: this layer writes its own rows straight into the next
            # layer's input buffer, whose other rows arrive by broadcast
            nxt = None
            if ex is not None and l != nl - 1 and \
                    not self.transform_first(l + 1):
                nxt = ex.buffer(("h", l + 1), self.weights.layers[l].out_dim,
                                _torch_dtype(self.config.embed_dtype), "cuda")
            # every layer is queued before any metric is read back, so the
            # host never stalls the device between layers
            torch.cuda.nvtx.range_push(f"atlas layer {l}")
            y, collect, _ = self.layer(
                l, h, input_flag=flag, defer_metrics=True,
                host_out=host_out if l == nl - 1 else None,
                out=None if nxt is None else ex.own(nxt), pieces=pieces)
            torch.cuda.nvtx.range_pop()
            pending.append(collect)
            if keep_layers:
                outs.append(y)
            pieces = None
            if l != nl - 1:
                flag = self.out_flags.get(l)
                if flag is not None and self.world > 1:
                    self.allreduce_max(flag)
                if nxt is not None:
                    # the owners' pieces in ascending row order; the next
                    # layer folds each one in as soon as it lands
                    torch.cuda.nvtx.range_push(f"atlas exchange {l + 1}")
                    h, pieces = nxt, ex.start(nxt)
                    torch.cuda.nvtx.range_pop()
                elif self.world > 1 and not self.transform_first(l + 1):
                    h = self.gather(y)  # a subclass's own gather
                else:
                    # a transform-first next layer (or one rank) needs only
                    # this rank's rows: it exchanges its narrower z instead
                    h = y
        self.last_layers = outs
        if not metrics:
            return y, None
        return y, [collect() for collect in pending]


def z_pitch(cols: int) -> int:
    """Row pitch (f32 elements) of a transform-first z buffer: whole
    64-byte units, so a narrow z row never straddles more DRAM bursts than
    it needs."""
    return -(-cols // 16) * 16


def _load_graph(topology_path, in_degrees):
    from .storage import GraphCSR

    hdr, offsets, nbrs = read_topology_arrays(topology_path,
                                              nbr_dtype=np.uint32)
    indeg = np.asarray(in_degrees, dtype=np.int64)
    topo_bytes = offsets.nbytes + nbrs.nbytes
    return GraphCSR(hdr.num_vertices, hdr.num_edges, offsets, nbrs,
                    indeg), topo_bytes


def _graduation_order(layer) -> np.ndarray:
    """The layer's graduation order (every destination once), from the
    control plane's graduation log ([n, ids..] per sub-batch)."""
    from . import _native as N

    flat = layer.log(N.LOG_GRADUATED)
    keep = np.ones(flat.size, dtype=bool)
    i = 0
    while i < flat.size:  # drop the per-batch counts
        keep[i] = False
        i += 1 + int(flat[i])
    return flat[keep]


def _write_output(layer_dir, y, config, grad_order) -> int:
    """One layer's output to its layer directory, laid out exactly as the
    reference's writer stage lays it out (oocgnn/writer.py:40-115: f32
    rows, partition buffers of spill_buffer bytes filled in graduation
    order, each flush sorted by id), so the directory is byte-identical to
    the reference's. y goes D2H into pinned memory first (a pageable .cpu()
    runs at a few GB/s). A failed write leaves no partial directory
    (oocgnn/writer.py:119-121). Returns the spill bytes written."""
    import torch

    from .chunks import write_graduation_layout

    pinned = torch.empty(y.shape, dtype=torch.float32, pin_memory=True)
    pinned.copy_(y)
    layer_dir = Path(layer_dir)
    if layer_dir.exists():
        shutil.rmtree(layer_dir)
    try:
        return write_graduation_layout(layer_dir, pinned.numpy(), grad_order,
                                       config.partitions,
                                       config.spill_buffer)
    except BaseException:
        shutil.rmtree(layer_dir, ignore_errors=True)
        raise


def _read_input(layer_dir, config):
    """A layer directory on the device: with direct_io (the reference's
    O_DIRECT reader, oocgnn/directio.py) straight from storage into HBM
    (GPUDirect Storage, or the library's pinned-bounce stream), otherwise
    through the pinned host reader and one upload."""
    if config.direct_io:
        from .chunks import load_layer_device
        _, h, nbytes, delivery, _ = load_layer_device(layer_dir,
                                                      device=config.device)
        return h, nbytes, delivery
    _, rows, nbytes, delivery = load_layer_input(layer_dir)
    return _upload(rows), nbytes, delivery


def _upload(rows):
    import torch

    t = torch.from_numpy(rows)
    if t.dtype == torch.float64:
        t = t.float()
    return t.pin_memory().cuda(non_blocking=True)


def run_layer(topology_path, in_degrees: np.ndarray, input_dir, output_dir,
              weights: ModelWeights, layer_index: int,
              config: PipelineConfig, scratch_dir=None) -> LayerMetrics:
    """One layer (oocgnn/runtime.py:114-220) through the device engine."""
    t0 = time.perf_counter()
    config.validate()
    meta = read_layer_meta(input_dir)
    expect = weights.embedding_dim(layer_index)
    if meta.dim != expect:
        raise ConfigError(f"layer {layer_index} expects {expect}-wide rows, "
                          f"input holds {meta.dim}")
    graph, topo_bytes = _load_graph(topology_path, in_degrees)
    h, feat_bytes, delivery = _read_input(input_dir, config)
    # the graduation log fixes the output's spill layout
    eng = Engine(graph, weights, replace(config, record_log=True))
    try:
        y, m, layer = eng.layer(layer_index, h)
        order = _graduation_order(layer)
        layer.close()
    finally:
        eng.close()
    written = _write_output(Path(output_dir), y, config, order)
    m.feature_bytes_read = feat_bytes
    m.bytes_read += feat_bytes + topo_bytes
    m.bytes_written += written
    m.delivery_counts = delivery
    m.wall_seconds = time.perf_counter() - t0
    return m


def run_inference(graph_dir, weights, config: PipelineConfig, out_dir,
                  metrics_path=None) -> RunReport:
    """Every layer; embeddings stay in HBM between layers and each
    layer_l/ directory is written like the reference's
    (oocgnn/runtime.py:223-264)."""
    t0 = time.perf_counter()
    config.validate()
    graph_dir, out_dir = Path(graph_dir), Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    if not isinstance(weights, ModelWeights):
        weights = read_weights(weights)
    hdr_path = graph_dir / TOPOLOGY_FILE
    hdr, offsets, nbrs = read_topology_arrays(hdr_path, nbr_dtype=np.uint32)
    in_degrees = read_in_degrees(graph_dir / INDEGREE_FILE, hdr.num_vertices)
    features_dir = graph_dir / "features"
    weights.validate(read_layer_meta(features_dir).dim)
    from .storage import GraphCSR

    graph = GraphCSR(hdr.num_vertices, hdr.num_edges, offsets, nbrs,
                     in_degrees)
    topo_bytes = offsets.nbytes + nbrs.nbytes
    h, feat_bytes, delivery = _read_input(features_dir, config)
    # the graduation log fixes each output's spill layout
    eng = Engine(graph, weights, replace(config, record_log=True))
    layers = []
    prev_dir = None
    try:
        for l in range(len(weights.layers)):
            tl = time.perf_counter()
            y, m, layer = eng.layer(l, h)
            order = _graduation_order(layer)
            layer.close()
            layer_out = out_dir / f"layer_{l}"
            m.bytes_written += _write_output(layer_out, y, config, order)
            if l == 0:
                m.feature_bytes_read = feat_bytes
                m.bytes_read += feat_bytes + topo_bytes
                m.delivery_counts = delivery
            else:
                nb = y.element_size() * h.numel()
                m.feature_bytes_read = nb
                m.delivery_counts = np.ones(hdr.num_vertices, np.uint16)
            m.wall_seconds = time.perf_counter() - tl
            layers.append(m)
            if config.discard_intermediate and l > 0 and prev_dir:
                shutil.rmtree(prev_dir, ignore_errors=True)
            prev_dir = layer_out
            h = y
    finally:
        eng.close()
    report = RunReport(layers, out_dir, time.perf_counter() - t0)
    write_metrics_csv(metrics_path or out_dir / "metrics.csv", layers)
    return report


def final_layer_dir(out_dir) -> Path:
    cands = sorted((p for p in Path(out_dir).glob("layer_*") if p.is_dir()),
                   key=lambda p: int(p.name.split("_")[1]))
    if not cands:
        raise ConfigError(f"{out_dir}: no layer outputs found")
    return cands[-1]


@dataclass
class CompareReport:
    max_abs_err: float
    mean_abs_err: float
    argmax_mismatches: int
    rows: int
    tolerance: float

    @property
    def ok(self) -> bool:
        return (self.max_abs_err <= self.tolerance
                and self.argmax_mismatches == 0)


def compare_outputs(dir_a, dir_b, tolerance: float) -> CompareReport:
    a = load_layer_matrix(final_layer_dir(dir_a))
    b = load_layer_matrix(final_layer_dir(dir_b))
    if a.shape != b.shape:
        raise ConfigError(f"shape mismatch: {a.shape} vs {b.shape}")
    diff = np.abs(a.astype(np.float64) - b.astype(np.float64))
    return CompareReport(
        float(diff.max(initial=0.0)),
        float(diff.mean()) if diff.size else 0.0,
        int(np.count_nonzero(a.argmax(axis=1) != b.argmax(axis=1))),
        a.shape[0], tolerance)


def clone_config(config: PipelineConfig, **overrides) -> PipelineConfig:
    return replace(config, **overrides)


__all__ = ["PipelineConfig", "RunReport", "Engine", "run_layer",
           "run_inference", "write_metrics_csv", "final_layer_dir",
           "compare_outputs", "clone_config", "ModelKind"]
