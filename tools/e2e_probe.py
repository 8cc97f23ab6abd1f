"""Stage timings of the end-to-end path (diagnostic; not part of bench):
host enqueue time of each stage and device time between the events
recorded after each stage, for the bench's e2e loop."""

import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2605_09402_b200 import storage as S  # noqa: E402
from paper_2605_09402_b200.runtime import Engine, PipelineConfig  # noqa: E402


HOST_MS = {}


def _trace(cls, names):
    """accumulate host time spent inside cls.<name> (blocking calls show)"""
    for n in names:
        f = getattr(cls, n)

        def wrap(*a, _f=f, _n=n, **k):
            t = time.perf_counter()
            try:
                return _f(*a, **k)
            finally:
                HOST_MS[_n] = HOST_MS.get(_n, 0.0) + 1e3 * (
                    time.perf_counter() - t)
        setattr(cls, n, wrap)


def main(v=2_400_000, deg=26, dim=100, tile_mb=256):
    graph, feats = S.synthetic_in_memory("uniform", v, deg, dim, 7)
    w = S.random_weights(S.ModelKind.GCN, [dim, 128, 128, 47], 5)
    cfg = PipelineConfig(chunk_budget=8 << 20, hot_slots=v, backend="tcgen05",
                         stream_tile_bytes=tile_mb << 20)
    print("tile MB", tile_mb)
    eng = Engine(graph, w, cfg)
    pinned = torch.from_numpy(feats).pin_memory()
    pin_off = torch.from_numpy(graph.offsets).pin_memory()
    pin_nb = torch.from_numpy(
        graph.neighbors.astype(np.uint32).view(np.int32)).pin_memory()
    pin_deg = torch.from_numpy(
        graph.in_degrees.astype(np.uint32).view(np.int32)).pin_memory()
    host_out = torch.empty((v, 47), dtype=torch.float32).pin_memory()
    names = ["graph", "layer0", "layer1", "layer2", "d2h"]
    for it in range(4):
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        hs = [time.perf_counter()]
        evs[0].record()
        eng.update_graph(pin_off, pin_nb, pin_deg)
        evs[1].record()
        if SYNC_GRAPH:
            torch.cuda.synchronize()
        hs.append(time.perf_counter())
        h = pinned
        pend = []
        for l in range(3):
            y, collect, _ = eng.layer(
                l, h, defer_metrics=True,
                host_out=host_out if (l == 2 and SLICED) else None)
            pend.append(collect)
            evs[2 + l].record()
            hs.append(time.perf_counter())
            h = y
        if not SLICED:
            host_out.copy_(y, non_blocking=True)
        evs[5].record()
        hs.append(time.perf_counter())
        torch.cuda.synchronize()
        end = time.perf_counter()
        ms = [c() for c in pend]
        dev = [evs[i].elapsed_time(evs[i + 1]) for i in range(5)]
        host = [1e3 * (hs[i + 1] - hs[i]) for i in range(5)]
        print("  host ms in:", {k: round(x, 2) for k, x in HOST_MS.items()})
        HOST_MS.clear()
        print(f"iter {it}: total {1e3 * (end - hs[0]):.1f} ms | " + " | ".join(
            f"{n} host {a:.1f} dev {b:.1f}" for n, a, b in zip(names, host, dev))
            + " | " + " ".join(f"L{m.layer}: agg {m.agg_ms:.1f} ctl "
                               f"{m.control_ms:.1f} tr {m.transform_ms:.1f}"
                               for m in ms), flush=True)
    eng.close()


SYNC_GRAPH = False
from paper_2605_09402_b200 import engine as _E  # noqa: E402

_trace(_E.DeviceLayer, ["reset", "bind_graph", "run_streamed",
                        "accumulator_ptr"])
_trace(_E.DeviceGraph, ["update"])

if __name__ == "__main__":
    for SLICED, SYNC_GRAPH in ((True, False),):
        print("sliced D2H", SLICED, "sync after graph", SYNC_GRAPH)
        for mb in (sys.argv[1:] or ["256"]):
            main(tile_mb=int(mb))
