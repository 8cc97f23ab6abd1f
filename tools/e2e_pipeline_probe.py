"""Timeline of the pipelined end-to-end path (bench.pipelined_e2e):
two engines on two host threads / CUDA streams, each request's device
events (start, topology+CSC done, output on host) relative to one start
event, and host-side time per call. Diagnostic only."""

import sys
import threading
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2605_09402_b200 import storage as S  # noqa: E402
from paper_2605_09402_b200.runtime import Engine, PipelineConfig  # noqa: E402


STAGGER_MS = 19.0


def main(v=2_400_000, deg=26, dim=100, inflight=2, steps=6):
    graph, feats = S.synthetic_in_memory("uniform", v, deg, dim, 7)
    w = S.random_weights(S.ModelKind.GCN, [dim, 128, 128, 47], 5)
    cfg = PipelineConfig(chunk_budget=8 << 20, hot_slots=v, backend="tcgen05")
    pinned = torch.from_numpy(feats).pin_memory()
    pin_off = torch.from_numpy(graph.offsets).pin_memory()
    pin_nb = torch.from_numpy(
        graph.neighbors.astype(np.uint32).view(np.int32)).pin_memory()
    pin_deg = torch.from_numpy(
        graph.in_degrees.astype(np.uint32).view(np.int32)).pin_memory()
    engines = [Engine(graph, w, cfg) for _ in range(inflight)]
    outs = [torch.empty((v, 47), dtype=torch.float32).pin_memory()
            for _ in engines]
    streams = [torch.cuda.Stream() for _ in engines]
    for r in range(inflight):  # warm
        with torch.cuda.stream(streams[r]):
            engines[r].update_graph(pin_off, pin_nb, pin_deg)
            engines[r].infer(pinned, host_out=outs[r], metrics=False)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    recs = []

    def worker(r, n):
        with torch.cuda.stream(streams[r]):
            time.sleep(r * STAGGER_MS / 1e3)
            for i in range(n):
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                h = [time.perf_counter()]
                e[0].record()
                engines[r].update_graph(pin_off, pin_nb, pin_deg)
                e[1].record()
                h.append(time.perf_counter())
                engines[r].infer(pinned, host_out=outs[r], metrics=False)
                e[2].record()
                h.append(time.perf_counter())
                streams[r].synchronize()
                h.append(time.perf_counter())
                recs.append((r, i, e, h))

    t0.record()
    host0 = time.perf_counter()
    th = [threading.Thread(target=worker, args=(r, steps // inflight))
          for r in range(inflight)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - host0) * 1e3
    print(f"{steps} requests, {inflight} in flight: {wall:.1f} ms wall, "
          f"{wall / steps:.1f} ms per request")
    for r, i, e, h in sorted(recs, key=lambda x: t0.elapsed_time(x[2][0])):
        d = [t0.elapsed_time(x) for x in e]
        print(f"engine {r} req {i}: device start {d[0]:7.1f} graph done "
              f"{d[1]:7.1f} infer done {d[2]:7.1f} | host: graph call "
              f"{(h[1] - h[0]) * 1e3:5.1f} infer call {(h[2] - h[1]) * 1e3:5.1f}"
              f" wait {(h[3] - h[2]) * 1e3:5.1f} ms (start +"
              f"{(h[0] - host0) * 1e3:6.1f})")


if __name__ == "__main__":
    if len(sys.argv) > 2:
        STAGGER_MS = float(sys.argv[2])
    main(inflight=int(sys.argv[1]) if len(sys.argv) > 1 else 2, steps=12)
