"""Stage timings of the end-to-end path (diagnostic; not part of bench)."""

import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2605_09402_b200 import storage as S  # noqa: E402
from paper_2605_09402_b200.runtime import Engine, PipelineConfig  # noqa: E402


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


def main(v=2_400_000, deg=26, dim=100):
    graph, feats = S.synthetic_in_memory("uniform", v, deg, dim, 7)
    w = S.random_weights(S.ModelKind.GCN, [dim, 128, 128, 47], 5)
    cfg = PipelineConfig(chunk_budget=8 << 20, hot_slots=v, backend="tcgen05")
    eng = Engine(graph, w, cfg)
    pinned = torch.from_numpy(feats).pin_memory()
    pin_off = torch.from_numpy(graph.offsets).pin_memory()
    pin_nb = torch.from_numpy(
        graph.neighbors.astype(np.uint32).view(np.int32)).pin_memory()
    pin_deg = torch.from_numpy(
        graph.in_degrees.astype(np.uint32).view(np.int32)).pin_memory()
    xd = pinned.cuda()
    for it in range(3):
        a = t()
        eng.graph.update(pin_off, pin_nb, pin_deg)
        b = t()
        y0, m0, _ = eng.layer(0, pinned)
        c = t()
        y0r, m0r, _ = eng.layer(0, xd)
        d = t()
        x2 = pinned.cuda(non_blocking=True)
        e = t()
        y, ms = eng.infer(xd)
        f = t()
        out = y.cpu()
        g = t()
        print(f"iter {it}: graph_update {1e3*(b-a):.1f} ms | layer0 streamed "
              f"{1e3*(c-b):.1f} (agg {m0.agg_ms:.1f} ctl {m0.control_ms:.1f}"
              f" tr {m0.transform_ms:.1f}) | layer0 resident {1e3*(d-c):.1f} "
              f"(agg {m0r.agg_ms:.1f}) | H2D feats {1e3*(e-d):.1f} | infer "
              f"{1e3*(f-e):.1f} | D2H {1e3*(g-f):.1f}", flush=True)
        assert torch.equal(y0.cpu(), y0r.cpu())
    eng.close()


if __name__ == "__main__":
    main()
