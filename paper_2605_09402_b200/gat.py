"""GAT on the broadcast layer engine (BASELINE config 3, kernel plan K10).

The reference has no GAT (SURVEY.md §8c "parity
unpinned"), so this module defines the model the way SURVEY.md A.5 fixes it
and oracle/gat.py restates it in float64 (DGL GATConv semantics, the
reference oracle's layer conventions: ReLU between layers, heads
concatenated in hidden layers and averaged in the last, zero in-degree ->
bias, no added self-loops, LeakyReLU slope 0.2).

GAT transforms first, so each layer is two device passes:

* pass A — ``z_ext = h . W_ext^T`` on the tcgen05 tensor cores
  (``atlas_transform_typed``; f16/bf16 inputs are exact in tf32). W_ext
  stacks W (H*F rows), then a_l[h]^T W_h and a_r[h]^T W_h, so the GEMM
  emits el and er as extra columns of every z row (``ZLayout``).
* pass B — ``atlas_layer_run_gat``: the edge-softmax scatter-aggregate over
  the rank's destination range with bias / head concat + ReLU / head mean
  fused (csrc/gat.cu), and the layer's control plane (pending = in-degree,
  GCN rules; the reference chunk plan sized by the z row).

With G ranks, rank g computes z for its own rows only and the z rows are
all-gathered (NCCL) before pass B: the one exchange per layer.

Weights file: AWTS version 2 (the reference's v1 has no heads or attention
vectors, oocgnn/storage.py:49-50, :556-571): header ``<4sIBIf`` (magic,
version 2, kind 3, layers, negative slope), then per layer ``<III`` (in,
heads, head_dim) and f32 W (H*F x in), a_l (H x F), a_r (H x F), b (H*F).
"""

from __future__ import annotations

import os
import struct
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .chunks import chunk_rows as plan_rows
from .errors import (BadMagicError, ConfigError, InvariantError,
                     TruncatedFileError, VersionMismatchError)
from .memstore import MemoryBudget
from .orchestrator import metrics_from_device

GAT_KIND = 3
_HDR = struct.Struct("<4sIBIf")
_HDR_LAYER = struct.Struct("<III")


@dataclass
class GATLayerWeights:
    in_dim: int
    heads: int
    head_dim: int
    weight: np.ndarray   # (heads*head_dim, in_dim) f32
    attn_l: np.ndarray   # (heads, head_dim) f32
    attn_r: np.ndarray   # (heads, head_dim) f32
    bias: np.ndarray     # (heads*head_dim,) f32

    @property
    def hf(self) -> int:
        return self.heads * self.head_dim


@dataclass
class GATWeights:
    layers: list
    negative_slope: float = 0.2
    kind: int = GAT_KIND

    def validate(self, feature_dim=None) -> None:
        if not self.layers:
            raise InvariantError("model must have at least one layer")
        prev = feature_dim
        for i, lw in enumerate(self.layers):
            if lw.weight.shape != (lw.hf, lw.in_dim):
                raise InvariantError(f"layer {i}: weight shape mismatch")
            for name in ("attn_l", "attn_r"):
                if getattr(lw, name).shape != (lw.heads, lw.head_dim):
                    raise InvariantError(f"layer {i}: {name} shape mismatch")
            if lw.bias.shape != (lw.hf,):
                raise InvariantError(f"layer {i}: bias shape mismatch")
            if prev is not None and lw.in_dim != prev:
                raise InvariantError(
                    f"layer {i}: in_dim {lw.in_dim}, expected {prev}")
            prev = self.out_dim(i)

    def embedding_dim(self, layer_index: int) -> int:
        return self.layers[layer_index].in_dim

    def out_dim(self, layer_index: int) -> int:
        lw = self.layers[layer_index]
        return lw.head_dim if layer_index == len(self.layers) - 1 else lw.hf

    def oracle_layers(self):
        return [(lw.weight, lw.attn_l, lw.attn_r, lw.bias, lw.heads)
                for lw in self.layers]


def random_gat_weights(dims, heads: int, seed: int,
                       gain: float = 1.0) -> GATWeights:
    """Glorot-uniform like storage.random_weights. dims = [in, hidden...,
    out]: hidden widths are heads*head_dim (concatenated), the last layer
    has ``heads`` heads of width dims[-1] (averaged)."""
    if len(dims) < 2:
        raise ConfigError("need at least [input_dim, output_dim]")
    rng = np.random.default_rng(seed)
    layers = []
    for i, (w_in, w_out) in enumerate(zip(dims[:-1], dims[1:])):
        last = i == len(dims) - 2
        if not last and w_out % heads:
            raise ConfigError(f"hidden width {w_out} not divisible by "
                              f"{heads} heads")
        f = w_out if last else w_out // heads
        hf = heads * f
        lim = gain * np.sqrt(6.0 / (w_in + hf))
        w = rng.uniform(-lim, lim, (hf, w_in))
        alim = gain * np.sqrt(6.0 / (f + 1))
        al = rng.uniform(-alim, alim, (heads, f))
        ar = rng.uniform(-alim, alim, (heads, f))
        b = gain * rng.uniform(-0.1, 0.1, hf)
        layers.append(GATLayerWeights(
            w_in, heads, f, w.astype(np.float32), al.astype(np.float32),
            ar.astype(np.float32), b.astype(np.float32)))
    return GATWeights(layers)


def write_gat_weights(path, model: GATWeights) -> None:
    model.validate()
    parts = [_HDR.pack(b"AWTS", 2, GAT_KIND, len(model.layers),
                       float(model.negative_slope))]
    for lw in model.layers:
        parts.append(_HDR_LAYER.pack(lw.in_dim, lw.heads, lw.head_dim))
        for a in (lw.weight, lw.attn_l, lw.attn_r, lw.bias):
            parts.append(np.ascontiguousarray(a, "<f4").tobytes())
    Path(path).write_bytes(b"".join(parts))


def read_gat_weights(path) -> GATWeights:
    path = Path(path)
    data = path.read_bytes()
    if len(data) < _HDR.size:
        raise TruncatedFileError(f"{path}: header short")
    magic, ver, kind, nlayers, slope = _HDR.unpack_from(data)
    if magic != b"AWTS":
        raise BadMagicError(f"{path}: expected magic b'AWTS', found {magic!r}")
    if ver != 2 or kind != GAT_KIND:
        raise VersionMismatchError(
            f"{path}: not a GAT weights file (version {ver}, kind {kind})")
    pos, layers = _HDR.size, []
    for i in range(nlayers):
        if pos + _HDR_LAYER.size > len(data):
            raise TruncatedFileError(f"{path}: layer {i} header short")
        fin, h, f = _HDR_LAYER.unpack_from(data, pos)
        pos += _HDR_LAYER.size
        arrs = []
        for shape in ((h * f, fin), (h, f), (h, f), (h * f,)):
            n = int(np.prod(shape))
            if pos + 4 * n > len(data):
                raise TruncatedFileError(f"{path}: layer {i} payload short")
            arrs.append(np.frombuffer(data, "<f4", n, pos).reshape(shape)
                        .copy())
            pos += 4 * n
        layers.append(GATLayerWeights(fin, h, f, *arrs))
    model = GATWeights(layers, float(slope))
    model.validate()
    return model


@dataclass(frozen=True)
class ZLayout:
    """Column layout of a pass-A row: [z | el (H) | er (H) | pad]. Head h
    of z sits at columns [h*stride, h*stride + F) with stride = F rounded
    up to a whole 16-byte chunk (zero columns between), so every 16-byte
    chunk the aggregation loads belongs to one head."""

    heads: int
    head_dim: int
    itemsize: int

    @property
    def epc(self) -> int:
        return 16 // self.itemsize

    def _up(self, n: int) -> int:
        return -(-n // self.epc) * self.epc

    @property
    def head_stride(self) -> int:
        return self._up(self.head_dim)

    @property
    def el_col(self) -> int:
        return self.heads * self.head_stride

    @property
    def er_col(self) -> int:
        return self.el_col + self.heads

    @property
    def ncols(self) -> int:
        """columns pass A writes (z, el, er, chunk padding)"""
        return self._up(self.er_col + self.heads)

    @property
    def line_rows(self) -> bool:
        """f32 z of <= 128 columns: pass B moves only the z part of a source
        row and recomputes el from it (csrc/gat.cu gat_ring), so rows start
        on 128-byte lines and a z part costs whole DRAM lines, not a
        [z | el] straddle."""
        return self.itemsize == 4 and self.el_col <= 128

    @property
    def ldz(self) -> int:
        n = self.ncols
        return -(-n // 32) * 32 if self.line_rows else n


def extended_weight(lw: GATLayerWeights, layout: ZLayout) -> np.ndarray:
    """W_ext (ncols x in): the heads of W at their strided rows, then
    a_l[h]^T W_h and a_r[h]^T W_h, zero elsewhere (computed in float64,
    stored f32), so z_ext = h . W_ext^T carries z, el and er."""
    w = lw.weight.astype(np.float64).reshape(lw.heads, lw.head_dim, lw.in_dim)
    ext = np.zeros((layout.ncols, lw.in_dim), dtype=np.float64)
    for h in range(lw.heads):
        r = h * layout.head_stride
        ext[r:r + lw.head_dim] = w[h]
    ext[layout.el_col:layout.el_col + lw.heads] = np.einsum(
        "hf,hfk->hk", lw.attn_l.astype(np.float64), w)
    ext[layout.er_col:layout.er_col + lw.heads] = np.einsum(
        "hf,hfk->hk", lw.attn_r.astype(np.float64), w)
    return ext.astype(np.float32)


def _torch_dtype(name):
    import torch

    return {"f32": torch.float32, "f16": torch.float16,
            "bf16": torch.bfloat16}[name]


def _reference_row_dtype(layer_index, x) -> str:
    """Row format a layer's input has in the reference's layer directories
    (what plan_chunks sizes chunks by, oocgnn/chunks.py:36-48): the dataset
    dtype for layer 0 (2-byte features plan as f16), f32 afterwards
    (oocgnn/writer.py:60-62 always writes f32)."""
    import torch

    if layer_index > 0:
        return "f32"
    return "f32" if x.dtype == torch.float32 else "f16"


class GATEngine:
    """Device-resident GAT inference over one destination range (the GAT
    counterpart of runtime.Engine; same PipelineConfig knobs).
    ``config.embed_dtype`` is the storage type of z and of the hidden
    layers' outputs (f32 default)."""

    def __init__(self, graph, weights: GATWeights, config, *, rank: int = 0,
                 world: int = 1, dist_group=None):
        import torch

        from .compute import device_code, get_backend
        from .engine import DeviceGraph
        from .storage import partition_ranges

        config.validate()
        weights.validate()
        self.config, self.weights = config, weights
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
        code = device_code(get_backend(config.backend or "tcgen05"))
        if code != 1:
            raise ConfigError("GAT pass A runs on the tcgen05 backend")
        self.zt = _torch_dtype(config.embed_dtype)
        item = torch.empty(0, dtype=self.zt).element_size()
        self.layouts, self.w_ext, self.zero_b, self.bias = [], [], [], []
        self.attn_l = []  # a_l at the strided z columns (line_rows layouts)
        # pass A with er fused into the GEMM epilogue (atlas_transform_er):
        # W is just the z rows, so 4 x 32 heads stay at n = 128 and on the
        # register-split / f16 kernels (W_ext's 136 rows did not)
        self.w_z, self.attn_r = [], []
        fuse_er = os.environ.get("ATLAS_GAT_ER", "1") != "0"
        for lw in weights.layers:
            lay = ZLayout(lw.heads, lw.head_dim, item)
            self.layouts.append(lay)
            self.w_ext.append(torch.as_tensor(extended_weight(lw, lay)).cuda())
            self.zero_b.append(torch.zeros(lay.ncols, device="cuda"))
            self.bias.append(torch.as_tensor(lw.bias).cuda())
            al = None
            if lay.line_rows:
                al = np.zeros((lw.heads, lay.head_stride), dtype=np.float32)
                al[:, :lw.head_dim] = lw.attn_l
                al = torch.as_tensor(al.reshape(-1)).cuda()
            self.attn_l.append(al)
            ar = wz = None
            if (fuse_er and al is not None and lw.heads <= 8
                    and lay.head_stride % 16 == 0 and lay.el_col <= 128):
                ar = np.zeros((lw.heads, lay.head_stride), dtype=np.float32)
                ar[:, :lw.head_dim] = lw.attn_r
                ar = torch.as_tensor(ar.reshape(-1)).cuda()
                wz = self.w_ext[-1][:lay.el_col].contiguous()
            self.attn_r.append(ar)
            self.w_z.append(wz)
        self._layers = {}
        self.last_layers = []
        self.exchange = None
        if world > 1:
            from .exchange import RangeExchange
            self.exchange = RangeExchange(graph.num_vertices, self.ranges,
                                          rank, dist_group,
                                          config.exchange_pieces)

    def close(self):
        for layer in self._layers.values():
            layer.close()
        self._layers.clear()
        self.graph.close()

    def _device_layer(self, l, lay):
        from .engine import DeviceLayer
        from . import _native as N

        layer = self._layers.get(l)
        gv = getattr(self.graph, "version", 0)
        if layer is not None and layer.handle:
            if layer.graph_version == gv:
                layer.reset()
            else:
                layer.bind_graph(self.graph)
                layer.graph_version = gv
            return layer
        cfg = self.config
        hf = lay.heads * lay.head_dim
        # a pending record is acc (H*F) + running max and sum per head
        rec = hf + 2 * lay.heads
        slots = (MemoryBudget(cfg.hot_slots, rec) if cfg.hot_slots else
                 MemoryBudget.from_bytes(cfg.hot_budget, rec)).slot_count
        layer = DeviceLayer(self.in_degrees, N.GAT, hf, hf, slots,
                            eviction=cfg.eviction, seed=cfg.seed,
                            evict_batch=cfg.evict_batch,
                            dst_range=(self.lo, self.hi),
                            record_log=cfg.record_log,
                            force_exact=cfg.force_exact, device=self.device)
        layer.graph_version = 0
        if gv:
            layer.bind_graph(self.graph)
            layer.graph_version = gv
        self._layers[l] = layer
        return layer

    def update_graph(self, offsets, neighbors, in_degrees):
        """Topology refresh (see runtime.Engine.update_graph)."""
        self.graph.update(offsets, neighbors, in_degrees)

    def gather(self, z_local):
        """All ranks' rows -> full tensor (owner broadcasts, in place)."""
        if self.world == 1:
            return z_local
        return self.exchange.gather(z_local, key=("in", z_local.shape[1],
                                                  z_local.dtype))

    def layer(self, l: int, h_local, defer_metrics: bool = False):
        """h_local: this rank's rows [lo, hi) of the layer input (CUDA
        tensor; layer 0 may pass the full feature matrix). Returns
        (y (nloc, out), metrics or a collector, device layer)."""
        import torch

        from .engine import transform_er, transform_typed

        w = self.weights
        lw, lay = w.layers[l], self.layouts[l]
        last = l == len(w.layers) - 1
        t0 = time.perf_counter()
        nloc = self.hi - self.lo
        if h_local.shape[0] == self.num_vertices and self.world > 1:
            h_local = h_local[self.lo:self.hi]
        if h_local.shape[1] != lw.in_dim:
            raise ConfigError(f"layer {l} expects {lw.in_dim}-wide rows, "
                              f"input holds {h_local.shape[1]}")
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        ex = self.exchange
        if ex is not None:
            # pass A writes this rank's z rows straight into its slice of
            # the exchange buffer; the owners' broadcasts fill the rest
            zfull = ex.buffer(("z", l), lay.ldz, self.zt, "cuda")
            z_local = ex.own(zfull)
        else:
            z_local = torch.empty((h_local.shape[0], lay.ldz), dtype=self.zt,
                                  device="cuda")
        if h_local.shape[0] and self.w_z[l] is not None and \
                h_local.dtype in (torch.float32, torch.float16):
            # z columns and er; el stays unwritten (gat_ring recomputes it
            # per edge from the z row it loads)
            transform_er(h_local, self.w_z[l], self.zero_b[l], z_local,
                         lay.el_col, self.attn_r[l], lay.er_col, lw.heads,
                         lay.head_stride)
        elif h_local.shape[0]:
            transform_typed(h_local, self.w_ext[l], self.zero_b[l], False,
                            z_local[:, :lay.ncols], 1)
        ev[1].record()
        if ex is not None:
            _, events = ex.start(zfull)
            ex.finish(events)
            z = zfull
        else:
            z = z_local
        # the control plane's chunk plan follows the layer INPUT's format
        # (in_dim rows; layer 0 in the dataset dtype, later layers f32 as
        # the reference writer emits them), never the z storage layout, so
        # pending / eviction / span integers depend only on model and graph
        rows = plan_rows(self.num_vertices, lw.in_dim,
                         _reference_row_dtype(l, h_local),
                         self.config.chunk_budget)
        layer = self._device_layer(l, lay)
        out_dim = lw.head_dim if last else lw.hf
        yt = torch.float32 if last else self.zt
        # 16-byte row pitch: the next layer's pass A reads y through TMA
        pitch = -(-out_dim // 8) * 8
        y = torch.empty((nloc, pitch), dtype=yt, device="cuda")[:, :out_dim]
        layer.run_gat(self.graph, z, lay, self.bias[l], y, mean_heads=last,
                      relu=not last, chunk_rows=rows,
                      negative_slope=w.negative_slope,
                      attn_l=self.attn_l[l])

        def collect():
            m = metrics_from_device(layer, l)
            m.agg_ms, m.control_ms = layer.timing()
            m.transform_ms = ev[0].elapsed_time(ev[1])
            m.gpu_seconds = time.perf_counter() - t0
            return m

        if defer_metrics:
            return y, collect, layer
        return y, collect(), layer

    def infer(self, x, keep_layers: bool = False, host_out=None,
              metrics: bool = True):
        """All layers; x is the full (V, in) feature matrix (device, or
        pinned host). Returns (final local output, [LayerMetrics]);
        ``host_out`` (pinned) also receives the final output."""
        import torch

        pending, outs = [], []
        h = x
        if not x.is_cuda:  # host (pinned) features: one H2D copy
            lo, hi = (self.lo, self.hi) if self.world > 1 else (0, x.shape[0])
            h = torch.empty((hi - lo, x.shape[1]), dtype=x.dtype,
                            device="cuda")
            h.copy_(x[lo:hi], non_blocking=True)
        for l in range(len(self.weights.layers)):
            y, collect, _ = self.layer(l, h, defer_metrics=True)
            pending.append(collect)
            if keep_layers:
                outs.append(y)
            h = y
        if host_out is not None:
            host_out.copy_(y, non_blocking=True)
        self.last_layers = outs
        if not metrics:
            return y, None
        return y, [collect() for collect in pending]


__all__ = ["GATLayerWeights", "GATWeights", "random_gat_weights",
           "write_gat_weights", "read_gat_weights", "ZLayout",
           "extended_weight", "GATEngine"]
