"""Exact control-plane replay under eviction pressure (diagnostic):
per-layer control-stream time and eviction counts of a resident pass with
a hot budget below the live set (min-pending eviction fires on every
chunk). ATLAS_SWEEP=0 selects the per-element machine instead of the sweep.
Usage: replay_probe.py V DEG DIM HOT_FRAC [MODEL]"""

import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2605_09402_b200 import storage as S  # noqa: E402
from paper_2605_09402_b200.runtime import Engine, PipelineConfig  # noqa: E402


def main():
    v, deg, dim = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    frac = float(sys.argv[4])
    model = sys.argv[5] if len(sys.argv) > 5 else "GCN"
    t = time.perf_counter()
    graph, feats = S.synthetic_in_memory("uniform", v, deg, dim, 7)
    print(f"generated V={v} E={graph.num_edges} in "
          f"{time.perf_counter() - t:.1f} s", flush=True)
    w = S.random_weights(S.ModelKind[model], [dim, 128, 47], 5)
    cfg = PipelineConfig(chunk_budget=8 << 20, hot_slots=max(1, int(v * frac)),
                         backend="tcgen05")
    eng = Engine(graph, w, cfg)
    x = torch.as_tensor(feats).cuda()
    for it in range(2):
        t = time.perf_counter()
        _, ms = eng.infer(x)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t
        print(f"iter {it}: wall {wall:.2f} s | " + " | ".join(
            f"L{m.layer} ctl {m.control_ms:.1f} ms agg {m.agg_ms:.1f} ms "
            f"fast {m.fast_path} evictions {m.evictions} reloads {m.reloads} "
            f"unique {m.unique_reloads} peak {m.hot_peak} "
            f"reload% {m.mean_reload_pct:.6f}"
            for m in ms), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
