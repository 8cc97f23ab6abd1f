#!/usr/bin/env python
"""Benchmark: full-graph layer-wise GNN inference, edges/s per layer.

Workload (BASELINE.json configs[1]): 3-layer GCN, dims [100,128,128,47],
on a synthetic ogbn-products-shaped uniform graph (V=2,400,000, avg degree
26 -> E=62,399,647, 100-d f32 features, seed 7; Glorot weights seed 5),
reference chunk plan of 8 MiB (115 chunks at layer 1), hot_slots = V.
A step is one full 3-layer inference; ``value`` = 3*E / step time
(edges/s per layer, summed over all ranks' destination ranges).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N>1 runs under torchrun: rank g owns partition_ranges(V, N)[g] and layer
outputs are exchanged with an NCCL all-gather (strong scaling: the graph
is fixed). ``--impl reference`` times the reference algorithm's CPU
restatement (oracle/engine.py, pinned bit-exactly to the reference) on a
bounded sample of the same workload on the host cores.
"""

import argparse
import gc
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

V, DEG, DIM, SEED, WSEED = 2_400_000, 26, 100, 7, 5
DIMS = [100, 128, 128, 47]
CHUNK_BUDGET = 8 << 20
METRIC = "full-graph inference edges/sec/layer"
WORKLOAD = ("cfg2: 3-layer GCN [100,128,128,47], synthetic uniform graph "
            "V=2,400,000 E=62,399,647 (avg degree 26, seed 7), 100-d f32 "
            "features, 8 MiB reference chunk plan (115 chunks), hot_slots=V")

# extra (non-default) workloads: IGB-Medium-shaped graph of BASELINE
# configs[2] (10M vertices, avg degree 12 -> ~120M edges, 1024-d f16
# features). Graph and features are generated on the device (torch
# Philox, seeded) -- the reference's numpy generator would take minutes at
# this size; parity is pinned on the small golden cases instead.
IGB_V, IGB_DEG, IGB_DIM = 10_000_000, 12, 1024
EXTRA = {
    "igb-medium-sage": ("SAGE", [1024, 128, 128, 19]),
    "igb-medium-gcn": ("GCN", [1024, 128, 128, 19]),
    # BASELINE configs[2] itself: 3-layer GAT, 4 heads x 32 (hidden 128)
    "igb-medium-gat": ("GAT", [1024, 128, 128, 19]),
}
GAT_HEADS = 4

# the north-star target (BASELINE configs[4], IGB-Large: 100M vertices,
# ~1.2B edges, 1024-d f16, 3-layer SAGE) on 8 GPUs, measured as ONE rank's
# share on one B200: destinations [0, 12.5M), its ~150M in-edges from all
# 100M sources, its 12.5M own feature rows (25.6 GB) streamed from pinned
# host memory. The other ranks' rows of every all-gathered tensor are
# stand-ins filled once outside the timed region; the NVLink all-gather
# bytes are reported, not timed.
# BASELINE configs[3] likewise: the ogbn-papers100M-shaped graph (111M
# vertices, avg degree 15 -> ~1.67B edges; the generator takes integer
# degrees, 15 is the nearer to 1.6B), 128-d f16, 3-layer SAGE
# [128,128,128,172], rank 0 of 8.
# name -> (model, dims, V, avg degree, feature dim, hot-slot fraction of
# the rank's range)
LARGE_G = 8
SLICE = {
    "igb-large-sage-rank0of8": ("SAGE", [1024, 128, 128, 19], 100_000_000,
                                12, 1024, 1.0),
    # the same with a hot budget of 10 % of the range: min-pending eviction
    # fires on every chunk and the control plane replays it exactly
    "igb-large-sage-rank0of8-evict": ("SAGE", [1024, 128, 128, 19],
                                      100_000_000, 12, 1024, 0.1),
    "papers100m-sage-rank0of8": ("SAGE", [128, 128, 128, 172], 111_000_000,
                                 15, 128, 1.0),
}


def build_inputs():
    from paper_2605_09402_b200 import storage as S

    graph, feats = S.synthetic_in_memory("uniform", V, DEG, DIM, SEED)
    weights = S.random_weights(S.ModelKind.GCN, DIMS, WSEED)
    return graph, feats, weights


def build_igb(kind, dims, seed=SEED):
    """Uniform random graph with the reference's semantics (multi-edges
    removed, self loops kept, CSR rows ascending) and U[-1,1) f16
    features, generated on cuda:0."""
    import torch

    from paper_2605_09402_b200 import storage as S

    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    m = IGB_V * IGB_DEG
    src = torch.randint(0, IGB_V, (m,), generator=gen, device="cuda")
    dst = torch.randint(0, IGB_V, (m,), generator=gen, device="cuda")
    key = torch.unique(src * IGB_V + dst)
    del src, dst
    s, t = key // IGB_V, key % IGB_V
    del key
    offsets = torch.zeros(IGB_V + 1, dtype=torch.int64, device="cuda")
    offsets[1:] = torch.cumsum(torch.bincount(s, minlength=IGB_V), 0)
    indeg = torch.bincount(t, minlength=IGB_V)
    graph = S.GraphCSR(IGB_V, int(t.numel()), offsets.cpu().numpy(),
                       t.to(torch.int32).cpu().numpy().view(np.uint32),
                       indeg.cpu().numpy())
    del s, t, offsets, indeg
    feats = torch.empty((IGB_V, IGB_DIM), dtype=torch.float16, device="cuda")
    feats.uniform_(-1.0, 1.0, generator=gen)
    if kind == "GAT":
        from paper_2605_09402_b200.gat import random_gat_weights
        return graph, feats, random_gat_weights(dims, GAT_HEADS, WSEED)
    weights = S.random_weights(S.ModelKind[kind], dims, WSEED)
    return graph, feats, weights


def build_large_slice(kind, dims, big_v, deg, dim, seed=SEED):
    """Rank 0's edges of a uniform graph of big_v vertices: the E/G edges
    whose destination is in [0, V/G), sources over all V (generated on the
    device; multi-edges removed, rows ascending)."""
    import torch

    from paper_2605_09402_b200 import storage as S

    lo, hi = S.partition_ranges(big_v, LARGE_G)[0]
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    m = big_v * deg // LARGE_G
    src = torch.randint(0, big_v, (m,), generator=gen, device="cuda")
    dst = torch.randint(lo, hi, (m,), generator=gen, device="cuda")
    key = torch.unique(src * hi + dst)
    del src, dst
    s, t = key // hi, key % hi
    del key
    offsets = torch.zeros(big_v + 1, dtype=torch.int64, device="cuda")
    offsets[1:] = torch.cumsum(torch.bincount(s, minlength=big_v), 0)
    indeg = torch.bincount(t, minlength=big_v)
    graph = S.GraphCSR(big_v, int(t.numel()), offsets.cpu().numpy(),
                       t.to(torch.int32).cpu().numpy().view(np.uint32),
                       indeg.cpu().numpy())
    del s, t, offsets, indeg
    own = torch.empty((hi - lo, dim), dtype=torch.float16, device="cuda")
    own.uniform_(-1.0, 1.0, generator=gen)
    feats = own.cpu().pin_memory()
    del own
    torch.cuda.empty_cache()
    weights = S.random_weights(S.ModelKind[kind], dims, WSEED)
    return graph, feats, weights


def slice_engine_class():
    from paper_2605_09402_b200.runtime import Engine

    class SliceEngine(Engine):
        """Rank 0 of G on one GPU: the other ranks' rows of each gathered
        tensor are stand-ins (filled once), the own block is copied in."""

        def __init__(self, *a, **k):
            super().__init__(*a, **k)
            self.exchange = None  # one GPU: no peers to broadcast with

        def gather(self, y_local):
            import torch

            if not hasattr(self, "_full"):
                self._full, self.remote_bytes = {}, 0
            key = (y_local.shape[1], y_local.dtype)
            full = self._full.get(key)
            if full is None:
                full = torch.empty((self.num_vertices, y_local.shape[1]),
                                   dtype=y_local.dtype, device="cuda")
                full.uniform_(-1.0, 1.0)
                self._full[key] = full
            full[self.lo:self.hi].copy_(y_local)
            self.remote_bytes += (self.num_vertices - (self.hi - self.lo)) \
                * y_local.shape[1] * y_local.element_size()
            return full

        def allreduce_max(self, t):
            pass

    return SliceEngine


def run_slice(args):
    """The igb-large rank slice (see SLICE): value = this rank's edges per
    second per layer; the projected 8-GPU figure assumes every rank runs
    the same share concurrently (weak slice of a strong-scaled job)."""
    import torch

    from paper_2605_09402_b200 import _native as N
    from paper_2605_09402_b200.runtime import PipelineConfig

    kind, dims, big_v, deg, dim, hot_frac = SLICE[args.workload]
    t_gen = time.perf_counter()
    graph, feats, weights = build_large_slice(kind, dims, big_v, deg, dim)
    gen_s = time.perf_counter() - t_gen
    rng = -(-big_v // LARGE_G)
    cfg = PipelineConfig(chunk_budget=CHUNK_BUDGET,
                         hot_slots=max(1, int(rng * hot_frac)),
                         backend=args.backend, embed_dtype=args.embed_dtype)
    eng = slice_engine_class()(graph, weights, cfg, rank=0, world=LARGE_G)
    for _ in range(args.warmup):
        eng.infer(feats)
    torch.cuda.synchronize()
    eng.remote_bytes = 0
    clocks = ClockSampler(0)
    clocks.start()
    launches0 = N.kernel_launches()
    start, stop = torch.cuda.Event(True), torch.cuda.Event(True)
    gc.disable()
    start.record()
    for _ in range(args.steps):
        eng.infer(feats, metrics=False)
    stop.record()
    torch.cuda.synchronize()
    gc.enable()
    launches = N.kernel_launches() - launches0
    clk = clocks.stop()
    ms = start.elapsed_time(stop) / args.steps
    remote = eng.remote_bytes / args.steps
    # one more step with its metrics taken at once (every layer's verdict
    # and, under eviction, its exact replay inside this wall-clock window)
    t_m = time.perf_counter()
    _, metrics = eng.infer(feats)
    torch.cuda.synchronize()
    metrics_wall = time.perf_counter() - t_m
    e_rank = graph.num_edges
    nl = len(weights.layers)
    h2d = feats.numel() * feats.element_size()
    print(json.dumps({
        "metric": METRIC + " (one rank of 8: weak slice of the 8-GPU job)",
        "value": nl * e_rank / (ms / 1e3), "unit": "edges/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": f"f16 in / f32 accumulate / {args.embed_dtype} embeddings",
        "data": "synthetic",
        "config": {"workload": f"{args.workload}: 3-layer {kind} {dims} on "
                   f"rank 0 of {LARGE_G} of a uniform graph V={big_v:,}, "
                   f"avg degree {deg} (rank edges {e_rank:,}), "
                   f"{dim}-d f16 own feature rows streamed from pinned host, "
                   f"hot_slots={cfg.hot_slots:,} ({hot_frac:.0%} of the "
                   "range)",
                   "parallelism": f"dst-range rank 0/{LARGE_G}",
                   "transform_backend": args.backend},
        "per_layer": [{"layer": m.layer, "agg_ms": round(m.agg_ms, 3),
                       "control_ms": round(m.control_ms, 3),
                       "transform_ms": round(m.transform_ms, 3),
                       "fast_path": m.fast_path, "messages": m.messages,
                       "evictions": m.evictions, "reloads": m.reloads}
                      for m in metrics],
        "ingest": {"h2d_bytes_per_step": h2d,
                   "gb_per_s_if_ingest_bound": h2d / (ms / 1e3) / 1e9},
        "allgather_bytes_received_per_step": remote,
        "projected_8gpu_edges_per_s_excluding_allgather":
            LARGE_G * nl * e_rank / (ms / 1e3),
        "step_with_metrics_wall_s": metrics_wall,
        "gpu_launches": launches, "clocks": clk, "generate_s": gen_s}),
        flush=True)
    eng.close()


def gat_agg_bytes(graph, weights, layouts, rank_range, zsize):
    """GAT pass B per layer: per in-edge the source's z part (H*F) and,
    unless el is recomputed from z (line-aligned f32 rows, gat_ring), its
    el sector (32 B), its u32 id; per destination CSC/degree (12 B), its
    er sector, and the output row written once."""
    lo, hi = rank_range
    e_g, v_g = int(graph.offsets[-1]), hi - lo
    out = []
    for l, (lw, lay) in enumerate(zip(weights.layers, layouts)):
        last = l == len(weights.layers) - 1
        osz = 4 if last else zsize
        el = 0 if lay.line_rows else 32
        out.append(e_g * (lw.hf * zsize + el) + 4 * e_g + 12 * v_g
                   + 32 * v_g + v_g * weights.out_dim(l) * osz)
    return out


def transform_roofline(weights, eng, per_layer, in_sizes, peaks, nloc,
                       nrows):
    """The dense transform per layer (tcgen05 GEMM): algorithmic HBM bytes
    (input rows once, output rows once, W once) and flops 2*rows*K*N over
    the layer's measured transform time. Aggregate-first: the f32 records
    (nloc x agg_dim) -> out. Transform-first: the layer input (all rows)
    -> z (npad per half, f32)."""
    out = []
    for l, lw in enumerate(weights.layers):
        t_ms = statistics.mean(step[l].transform_ms for step in per_layer)
        last = l == len(weights.layers) - 1
        if getattr(eng, "transform_first", lambda _: False)(l):
            k = weights.embedding_dim(l)
            npad = -(-lw.out_dim // 4) * 4
            n = npad * (2 if weights.kind == 1 else 1)
            rows = nrows
            b = rows * k * in_sizes[l] + rows * n * 4 + n * k * 4
        else:
            k, n = weights.agg_dim(l), lw.out_dim
            rows = nloc
            osz = 4 if last else in_sizes[min(l + 1, len(in_sizes) - 1)]
            b = rows * k * 4 + rows * n * osz + n * k * 4
        fl = 2.0 * rows * k * n
        gbs = b / (t_ms / 1e3) / 1e9 if t_ms > 0 else None
        out.append({"layer": l, "rows": rows, "k": k, "n": n,
                    "ms": round(t_ms, 3), "bytes": b,
                    "hbm_gbs": gbs and round(gbs, 1),
                    "hbm_frac": gbs and round(gbs / peaks["hbm_gbs"], 3),
                    "tflops": t_ms and round(fl / (t_ms / 1e3) / 1e12, 1)})
    return {"bound": "hbm", "note": "3xTF32 (f32 input) or hi/lo f16 "
            "(f16 input) on tcgen05; intensity <= 64 flop/B, below the "
            "ridge, so HBM bytes are the roofline", "layers": out}


def agg_bytes(graph, weights, rank_range, in_sizes, eng=None, out_size=4):
    """Algorithmic HBM bytes of the resident scatter-aggregate per layer
    (DESIGN.md §4): gather every in-edge's source row once (the layer
    input does not fit in L2), read the u32 source id per edge and the
    CSC/in-degree arrays per destination, read the destination's own row
    for the SAGE/GIN self term, write each f32 record once. A
    transform-first layer (eng.transform_first(l)) gathers z rows of
    npad f32 instead and writes the layer output directly."""
    lo, hi = rank_range
    e_g = int(graph.offsets[-1]) if (lo, hi) == (0, graph.num_vertices) \
        else int(np.count_nonzero((graph.neighbors >= lo)
                                  & (graph.neighbors < hi)))
    v_g = hi - lo
    self_row = weights.kind != 0
    out = []
    for l, lw in enumerate(weights.layers):
        d, s = weights.embedding_dim(l), in_sizes[l]
        if eng is not None and eng.transform_first(l):
            npad = -(-lw.out_dim // 4) * 4
            out.append(e_g * npad * 4 + 4 * e_g + 12 * v_g
                       + (v_g * npad * 4 if self_row else 0)
                       + v_g * lw.out_dim * out_size)
            continue
        out.append(e_g * d * s + 4 * e_g + 12 * v_g
                   + (v_g * d * s if self_row else 0)
                   + 4 * weights.agg_dim(l) * v_g)
    return out


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled through NVML from
    a thread during the timed region (no subprocess: forking a process that
    maps tens of GB stalls the launching thread)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, device, period=0.01):
        self.device, self.period = device, period
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self.nv = None

    def start(self):
        if os.environ.get("ATLAS_BENCH_NO_NVML"):  # diagnostics only
            return
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h,
                                                        nv.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - no NVML: report n/a
            self.nv = None
            return
        self.done = threading.Event()
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def reset(self):
        """Drop the samples taken so far (before the timed region)."""
        self.sm, self.reasons = [], set()

    def _sample(self):
        nv = self.nv
        self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        for name, attr in self.REASONS:
            if mask & getattr(nv, attr, 0):
                self.reasons.add(name)

    def _run(self):
        while not self.done.is_set():
            try:
                self._sample()
            except Exception:  # noqa: BLE001
                break
            self.done.wait(self.period)

    def stop(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["n/a"]}
        self.done.set()
        self.thread.join(timeout=2)
        if not self.sm:
            self._sample()
        return {"sm_mhz": statistics.median(self.sm),
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml"}


def cpu_baseline(graph, feats, weights, seconds=20.0):
    """Reference algorithm (oracle/engine.py) on the first chunks of layer
    1, process_chunk only, single thread; edges/s extrapolates linearly
    (the paper's own method)."""
    from oracle import engine as OE

    rows = max(1, CHUNK_BUDGET // (DIM * 4))
    layer = OE.Layer(graph.in_degrees, OE.GCN, DIM, DIM, graph.num_vertices)
    t0 = time.perf_counter()
    edges = chunks = 0
    for start in range(0, graph.num_vertices, rows):
        end = min(start + rows, graph.num_vertices)
        lo, hi = int(graph.offsets[start]), int(graph.offsets[end])
        layer.process_chunk(start, end, feats[start:end],
                            graph.offsets[start:end + 1] - lo,
                            graph.neighbors[lo:hi])
        edges += hi - lo
        chunks += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    return {"value": edges / dt, "unit": "edges/s", "cores": 1,
            "kind": "port",
            "sample": f"layer 1, first {chunks} of "
                      f"{-(-graph.num_vertices // rows)} reference chunks "
                      f"({edges} edges, {dt:.1f} s), process_chunk "
                      f"(scatter-aggregate + pending/eviction control), "
                      f"numpy restatement pinned to the reference, 1 thread "
                      f"of {os.cpu_count()} host cores"}


def gat_cpu_baseline(graph, x, weights, seconds=15.0, block=50_000,
                     batch=2000):
    """The reference has no GAT, so there is no reference
    CPU path for configs[2]: this times this repo's float64 GAT oracle
    (oracle/gat.py ``gat_layer_at``, the CPU restatement the GPU is checked
    against) on layer 1, destination batch after batch over the first
    ``block`` destinations; edges/s extrapolates linearly like the
    reference arm. The in-edge lists and source rows are prepared once,
    outside the timed calls."""
    import torch

    from oracle import gat as OG

    lw = weights.layers[0]
    nbrs = np.asarray(graph.neighbors, dtype=np.int64)
    sel = np.flatnonzero(nbrs < block)
    src = np.searchsorted(graph.offsets, sel, side="right") - 1
    dst = nbrs[sel]
    order = np.lexsort((src, dst))
    src, dst = src[order], dst[order]
    offs = np.concatenate([[0], np.cumsum(np.bincount(dst,
                                                      minlength=block))])
    uniq, inv = np.unique(src, return_inverse=True)
    rows = x[torch.as_tensor(uniq).cuda()].cpu().numpy()
    own = x[:block].cpu().numpy()
    t0 = time.perf_counter()
    edges = done = 0
    while done < block and time.perf_counter() - t0 < seconds:
        b1 = min(block, done + batch)
        e0, e1 = offs[done], offs[b1]
        u, k = np.unique(inv[e0:e1], return_inverse=True)
        OG.gat_layer_at(np.arange(done, b1), offs[done:b1 + 1] - e0, k,
                        rows[u], own[done:b1], lw.weight, lw.attn_l,
                        lw.attn_r, lw.bias, lw.heads, concat=True)
        edges += e1 - e0
        done = b1
    dt = time.perf_counter() - t0
    return {"value": edges / dt, "unit": "edges/s", "cores": os.cpu_count(),
            "kind": "port",
            "sample": f"NO reference CPU path exists for GAT (the reference "
                      f"has none); this repo's float64 GAT oracle on layer 1 "
                      f"(1024 -> 4x32): destinations [0, {done}), {edges} "
                      f"in-edges in {dt:.1f} s, numpy + multi-threaded BLAS"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    graph, feats, weights = build_inputs()
    for _ in range(args.warmup):
        cpu_baseline(graph, feats, weights, seconds=2.0)
    vals = []
    for _ in range(args.steps):
        vals.append(cpu_baseline(graph, feats, weights, seconds=10.0))
    value = statistics.median(v["value"] for v in vals)
    cb = dict(vals[-1])
    cb["value"] = value
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "edges/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup,
        # one full step (3 layers over all E edges) at the sampled rate
        "ms_per_step": len(weights.layers) * graph.num_edges / value * 1e3,
        "ms_per_step_note": "extrapolated from the bounded samples",
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "parallelism": "host, 1 thread"},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


def pipelined_e2e(eng, Eng, graph, weights, cfg, pinned, pin_off, pin_nb,
                  pin_deg, y_ref, out_shape, steps, inflight, stagger_ms=0.0):
    """Whole-job e2e time per step with `inflight` requests in flight:
    request r runs on engine r % inflight (the measured engine plus clones
    with their own device buffers), each engine driven by its own host
    thread on its own stream. Returns ms per step (wall clock over all
    steps / steps), after checking every engine's output."""
    import threading

    import torch

    engines = [eng] + [Eng(graph, weights, cfg) for _ in range(inflight - 1)]
    outs = [torch.empty(out_shape, dtype=torch.float32).pin_memory()
            for _ in engines]
    streams = [torch.cuda.Stream() for _ in engines]
    per = [steps // inflight + (1 if r < steps % inflight else 0)
           for r in range(inflight)]
    go = threading.Barrier(inflight + 1)
    errs = []
    stagger_s = stagger_ms / 1e3

    def worker(r, n, warm):
        try:
            with torch.cuda.stream(streams[r]):
                if not warm:
                    go.wait()
                    # staggered start: request r's uploads overlap the
                    # layers of the requests ahead of it instead of all
                    # engines contending for the H2D engine in lockstep
                    time.sleep(r * stagger_s)
                for _ in range(n):
                    engines[r].update_graph(pin_off, pin_nb, pin_deg)
                    # metrics=False: no device-wide synchronisation (the
                    # layer metrics' finish would serialise the engines)
                    engines[r].infer(pinned, host_out=outs[r],
                                     metrics=False)
                    streams[r].synchronize()
        except Exception as e:  # noqa: BLE001 - reported by the caller
            errs.append(e)
            if not warm:
                go.abort()

    # warm every clone once (allocations, first-use paths), untimed
    for r in range(1, inflight):
        worker(r, 1, True)
    threads = [threading.Thread(target=worker, args=(r, per[r], False))
               for r in range(inflight)]
    for t in threads:
        t.start()
    torch.cuda.synchronize()
    go.wait()
    t0 = time.perf_counter()
    for t in threads:
        t.join()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    for e in engines[1:]:
        e.close()
    if errs:
        raise errs[0]
    want = y_ref.cpu()
    for r in range(inflight):
        if per[r]:
            assert torch.equal(outs[r], want), f"pipelined e2e output {r}"
    return wall / steps


def self_launch(n: int) -> int:
    """``bench.py --gpus N`` without a launcher: start N ranks with
    torch.distributed.run on 127.0.0.1 (NCCL inside), pass their output
    through, return the launcher's exit code."""
    import socket
    import subprocess

    import torch

    have = torch.cuda.device_count()
    if have < n:
        print(json.dumps({"error": f"--gpus {n} needs {n} visible GPUs, "
                          f"found {have}"}), flush=True)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.run(cmd, check=False).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="atlas")
    ap.add_argument("--backend", default="tcgen05")
    ap.add_argument("--workload", default="cfg2",
                    choices=["cfg2"] + sorted(EXTRA) + sorted(SLICE))
    ap.add_argument("--embed-dtype", default=None,
                    choices=["f32", "f16", "bf16"],
                    help="storage type of intermediate embeddings (GAT: "
                         "of z); f32 (default) keeps the reference's f32 "
                         "semantics; the 8-GPU rank slices default to f16 "
                         "(SURVEY.md §8d: layer inputs >= 2 are fp16 for "
                         "configs 4/5)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cfg3", action="store_true",
                    help="skip the IGB-Medium GAT (BASELINE configs[2]) "
                         "measurement the default cfg2 run nests as 'cfg3'")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-alt", action="store_true",
                    help="skip the bit-exact (stable) backend re-run")
    args = ap.parse_args()
    if args.embed_dtype is None:
        args.embed_dtype = "f16" if args.workload in SLICE else "f32"
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ \
            and args.impl != "reference":
        # one process per GPU: re-launch this script under torchrun
        sys.exit(self_launch(args.gpus))
    if args.impl == "reference":
        run_reference(args)
        return
    if args.workload in SLICE:
        run_slice(args)
        return

    import torch
    import torch.distributed as dist

    from paper_2605_09402_b200 import _native as N
    from paper_2605_09402_b200.runtime import Engine, PipelineConfig

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test knobs for exercising the N-rank path on a 1-GPU box: every rank
    # on cuda:0 and gloo collectives (the driver's N-GPU runs use neither)
    if os.environ.get("ATLAS_BENCH_SHARE_GPU") == "1":
        local = 0
    backend = os.environ.get("ATLAS_BENCH_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group(
                "nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    line = measure(args, world, rank, local)
    if line is not None and args.workload == "cfg2" and world == 1 \
            and not args.no_cfg3:
        # BASELINE configs[2] (IGB-Medium GAT), the largest single-GPU
        # config, measured in the same run and reported inside the line
        import copy
        gc.collect()
        torch.cuda.empty_cache()
        a3 = copy.copy(args)
        a3.workload, a3.no_alt = "igb-medium-gat", True
        line["cfg3"] = measure(a3, world, rank, local)
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def measure(args, world, rank, local):
    """One workload on this rank; rank 0 returns its JSON-line dict."""
    import torch
    import torch.distributed as dist

    from paper_2605_09402_b200 import _native as N
    from paper_2605_09402_b200.runtime import Engine, PipelineConfig

    t_gen = time.perf_counter()
    if args.workload == "cfg2":
        graph, feats, weights = build_inputs()
        x = torch.from_numpy(feats).cuda()
        workload, dtype = WORKLOAD, "f32"
        cfg = PipelineConfig(chunk_budget=CHUNK_BUDGET, hot_slots=V,
                             backend=args.backend, device=local,
                             embed_dtype=args.embed_dtype)
    else:
        kind, dims = EXTRA[args.workload]
        graph, x, weights = build_igb(kind, dims)
        feats = None
        workload = (f"{args.workload}: 3-layer {kind} {dims}, synthetic "
                    f"uniform graph V={IGB_V:,} E={graph.num_edges:,} (avg "
                    f"degree {IGB_DEG}, device Philox seed {SEED}), "
                    f"{IGB_DIM}-d f16 features, 8 MiB reference chunk plan, "
                    f"hot_slots=V")
        dtype = (f"f16 in / f32 accumulate / {args.embed_dtype} "
                 f"intermediate embeddings")
        cfg = PipelineConfig(chunk_budget=CHUNK_BUDGET, hot_slots=IGB_V,
                             backend=args.backend, device=local,
                             embed_dtype=args.embed_dtype)
    gen_s = time.perf_counter() - t_gen
    is_gat = args.workload.endswith("-gat")
    if is_gat:
        from paper_2605_09402_b200.gat import GATEngine
        dims = [weights.embedding_dim(0)] + [
            weights.out_dim(l) for l in range(len(weights.layers))]
        cfg.backend = "tcgen05"
        Eng = GATEngine
    else:
        dims = [weights.embedding_dim(0)] + [lw.out_dim
                                             for lw in weights.layers]
        Eng = Engine
    nlayers = len(weights.layers)
    t_setup = time.perf_counter()
    eng = Eng(graph, weights, cfg, rank=rank, world=world)
    setup_s = time.perf_counter() - t_setup

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    # the NVML sampler thread starts (and takes its first samples) during
    # the warm-up; only samples from the timed region are kept
    clocks = ClockSampler(local)
    clocks.start()
    # the warm-up holds each step's output while the next one runs, as the
    # timed loop does, so the caching allocator owns both output buffers
    # before timing (otherwise the 2nd timed step pays a cudaMalloc)
    y = None
    for _ in range(args.warmup):
        y, _ = eng.infer(x)
    barrier()
    clocks.reset()
    if eng.exchange is not None:
        eng.exchange.bytes_received = 0
    launches0 = N.kernel_launches()
    start, stop = torch.cuda.Event(True), torch.cuda.Event(True)
    marks = [torch.cuda.Event(True) for _ in range(args.steps)]
    per_layer = []
    # steps are queued back to back (the host never waits for the device
    # inside the timed region); the last step's metrics are read after it
    gc.disable()
    start.record()
    for i in range(args.steps):
        y, _ = eng.infer(x, metrics=False)
        marks[i].record()
    stop.record()
    barrier()
    gc.enable()
    launches = N.kernel_launches() - launches0
    clk = clocks.stop()
    exchange = None
    if eng.exchange is not None:
        exchange = {
            "kind": "owner broadcasts (NCCL) into each layer's input "
                    "buffer, folded in piece by piece",
            "pieces_per_rank": eng.exchange.pieces_per_rank,
            "bytes_received_per_step_rank0":
                eng.exchange.bytes_received / args.steps}
    # one more (untimed) step with its metrics: per-layer kernel times from
    # CUDA events on the launching stream, and the integer counters
    y, metrics = eng.infer(x)
    per_layer.append(metrics)
    # the bit-exact transform backend (reference f32 operation order, every
    # embedding identical to the reference's), timed the same way
    alt = "stable" if (args.backend != "stable" and not args.no_alt
                       and not is_gat) else None
    alt_ms = None
    if alt:
        from paper_2605_09402_b200.compute import get_backend
        main_backend, eng.backend = eng.backend, get_backend(alt)
        eng.infer(x)
        barrier()
        a0, a1 = torch.cuda.Event(True), torch.cuda.Event(True)
        a0.record()
        for _ in range(args.steps):
            eng.infer(x, metrics=False)
        a1.record()
        barrier()
        alt_ms = a0.elapsed_time(a1) / args.steps
        eng.backend = main_backend
    ms = start.elapsed_time(stop) / args.steps
    step_ms = [round(start.elapsed_time(marks[0]), 3)] + [
        round(a.elapsed_time(b), 3) for a, b in zip(marks, marks[1:])]
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    edges = graph.num_edges
    value = nlayers * edges / (ms / 1e3)

    # roofline of the dominant kernel (scatter-aggregate), CUDA events
    in_sizes = [x.element_size()] + [
        {"f32": 4, "f16": 2, "bf16": 2}[cfg.embed_dtype]] * (nlayers - 1)
    if is_gat:
        per_b = gat_agg_bytes(graph, weights, eng.layouts, (eng.lo, eng.hi),
                              in_sizes[-1])
        kinds = ["gat_ring" if eng.layouts[l].line_rows else "gat_bulk"
                 for l in range(nlayers)]
    else:
        per_b = agg_bytes(graph, weights, (eng.lo, eng.hi), in_sizes, eng,
                          in_sizes[-1])

        def kind_of(l):
            if eng.transform_first(l):
                return "agg_tf_multi / agg_ring_epi (transform-first)"
            row = weights.embedding_dim(l) * in_sizes[l]
            return ("agg_bulk" if row > 512 else
                    "agg_ring" if row > 256 else "agg_sub_ring")
        kinds = [kind_of(l) for l in range(nlayers)]
    agg_b = sum(per_b)
    # dominant aggregation kernel: the kind with the most device time;
    # achieved = its algorithmic bytes / its mean launch time (CUDA events)
    groups = {}
    for l, k in enumerate(kinds):
        ms_l = statistics.mean(step[l].agg_ms for step in per_layer)
        g = groups.setdefault(k, [0, 0.0, 0])
        g[0] += per_b[l]
        g[1] += ms_l
        g[2] += 1
    dom = max(groups, key=lambda k: groups[k][1])
    dom_b, dom_ms, dom_n = groups[dom]
    achieved = dom_b / (dom_ms / 1e3) / 1e9
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {"hbm_gbs": 6650.0}
    traffic = None
    prof = ROOT / "profiles" / f"agg_traffic_{args.workload}.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get(dom)

    e2e_line = None
    if not args.no_e2e:
        # end to end through the public API with HOST buffers, every step:
        # topology H2D + CSC rebuild (atlas_graph_update), features
        # streamed H2D in double-buffered tiles overlapped with layer-1
        # aggregation (atlas_layer_run_streamed), all layers, output D2H
        pinned = (torch.from_numpy(feats) if feats is not None
                  else x.cpu()).pin_memory()
        pin_off = torch.from_numpy(graph.offsets).pin_memory()
        pin_nb = torch.from_numpy(np.ascontiguousarray(
            graph.neighbors, dtype=np.uint32).view(np.int32)).pin_memory()
        pin_deg = torch.from_numpy(np.ascontiguousarray(
            graph.in_degrees, dtype=np.uint32).view(np.int32)).pin_memory()
        host_out = torch.empty((eng.hi - eng.lo, dims[-1]),
                               dtype=torch.float32).pin_memory()
        e2e_ms = []
        for i in range(args.steps + 1):
            barrier()
            t0 = time.perf_counter()
            eng.update_graph(pin_off, pin_nb, pin_deg)
            yd, _ = eng.infer(pinned, host_out=host_out)
            torch.cuda.synchronize()
            if i:
                e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e_seq = statistics.median(e2e_ms)
        assert torch.equal(host_out, y.cpu()), "e2e output differs"
        # serving throughput: two requests in flight, each on its own
        # engine, host thread and CUDA stream, so one request's uploads
        # (H2D copy engine) overlap the other's layers and output download
        # (D2H engine); every step still uploads its topology and features
        # and downloads its output inside the timed region
        e2e_pipe = None
        inflight = int(os.environ.get("ATLAS_BENCH_INFLIGHT", "2"))
        if world == 1 and not is_gat and inflight > 1:
            # more requests than --steps: the staggered start is a ramp
            e2e_pipe = pipelined_e2e(eng, Eng, graph, weights, cfg, pinned,
                                     pin_off, pin_nb, pin_deg, y,
                                     host_out.shape, max(args.steps, 12),
                                     inflight, e2e_seq / inflight)
        e2e = e2e_pipe if e2e_pipe is not None else e2e_seq
        if world > 1:
            t = torch.tensor([e2e], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e = float(t.item())
        h2d = pinned.numel() * pinned.element_size() + graph.offsets.nbytes \
            + 4 * graph.num_edges + 4 * graph.num_vertices
        e2e_line = {"value": nlayers * edges / (e2e / 1e3),
                    "unit": "edges/s", "ms_per_step": e2e,
                    "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": host_out.numel() * 4,
                    "includes": "graph upload + CSC build, feature H2D, "
                                f"{nlayers} layers, output D2H",
                    "requests_in_flight": inflight if e2e_pipe else 1,
                    "requests": max(args.steps, 12) if e2e_pipe else
                    args.steps,
                    "sequential": {
                        "value": nlayers * edges / (e2e_seq / 1e3),
                        "ms_per_step": e2e_seq,
                        "note": "one request at a time: the host waits for "
                                "each output before uploading the next "
                                "request (latency)"}}
    if rank == 0:
        last = per_layer[-1]
        line = {
            "metric": METRIC, "value": value, "unit": "edges/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": workload,
                       "global_batch": graph.num_vertices,
                       "parallelism": f"dst-range x{world}",
                       "transform_backend": args.backend,
                       "l2": "inputs larger than L2 (layer inputs >= 0.96 "
                             "GB vs 126 MB), no flush"},
            "step_ms": step_ms,
            "per_layer_note": "agg_ms: launch-stream events around the "
                              "aggregation; control_ms: the control "
                              "stream's span, which runs concurrently "
                              "with the aggregation (not additive)",
            "per_layer_ms": [round(max(m.agg_ms, m.control_ms)
                                   + m.transform_ms, 3) for m in last],
            "per_layer": [{"layer": m.layer, "agg_ms": round(m.agg_ms, 3),
                           "control_ms": round(m.control_ms, 3),
                           "transform_ms": round(m.transform_ms, 3),
                           "fast_path": m.fast_path, "messages": m.messages,
                           "evictions": m.evictions, "hot_peak": m.hot_peak}
                          for m in last],
            "roofline": {"bound": "hbm", "achieved": achieved,
                         "model": "GAT" if is_gat else None,
                         "peak": peaks.get("hbm_gbs", 6650.0), "unit": "GB/s",
                         "frac": achieved / peaks.get("hbm_gbs", 6650.0),
                         "traffic": traffic,
                         "kernel": dom,
                         "launches_per_step": dom_n,
                         "algorithmic_bytes_per_launch": dom_b / dom_n,
                         "all_kernels": {
                             k: {"bytes": g[0], "ms": round(g[1], 3),
                                 "frac": g[0] / (g[1] / 1e3) / 1e9 /
                                 peaks.get("hbm_gbs", 6650.0)}
                             for k, g in groups.items()},
                         "algorithmic_bytes_per_step": agg_b},
            "transform": None if is_gat else transform_roofline(
                weights, eng, per_layer, in_sizes, peaks, eng.hi - eng.lo,
                graph.num_vertices),
            "e2e": e2e_line,
            "bit_exact_backend": None if alt is None else {
                "backend": alt, "ms_per_step": alt_ms,
                "value": nlayers * edges / (alt_ms / 1e3),
                "note": "every embedding bit-identical to the reference; "
                        "the headline backend is within the stated "
                        "tolerance (tests/test_gpu_parity.py)"},
            "gpu_launches": launches,
            "gpu_launches_per_step": launches / max(1, args.steps),
            "exchange": exchange,
            "clocks": clk,
            "setup_s": setup_s, "generate_s": gen_s,
        }
        if not args.no_cpu_baseline and world == 1:
            if feats is not None:
                line["cpu_baseline"] = cpu_baseline(graph, feats, weights)
            elif is_gat:
                line["cpu_baseline"] = gat_cpu_baseline(graph, x, weights)
    eng.close()
    return line if rank == 0 else None


if __name__ == "__main__":
    main()
