"""Register-split transform vs the shared-memory kernel on many shapes
(multi-tile persistent CTAs included). Prints the shapes that differ."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_09402_b200.engine import transform_typed  # noqa: E402


def run(x, w, b, y, env):
    for key in ("ATLAS_TRANSFORM_R", "ATLAS_TRANSFORM_T"):
        os.environ.pop(key, None)
    os.environ.update(env)
    transform_typed(x, w, b, True, y, 1)
    torch.cuda.synchronize()
    return y.float().clone()


bad = 0
for rows in (777, 40000, 300000):
    for k in (32, 36, 64, 96, 100, 128):
        for n in (16, 48, 120, 128):
            x = torch.randn(rows, k, device="cuda")
            w = torch.randn(n, k, device="cuda") / k ** 0.5
            b = torch.randn(n, device="cuda")
            y = torch.empty(rows, n, device="cuda")
            a = run(x, w, b, y, {"ATLAS_TRANSFORM_R": "0"})
            c = run(x, w, b, y, {})
            d = (a - c).abs().max().item()
            if d > 1e-5:
                bad += 1
                rr = ((a - c).abs().max(dim=1).values > 1e-5).nonzero()
                print(f"rows={rows} k={k} n={n}: max diff {d:.3e}, "
                      f"{rr.numel()} bad rows, first {rr[:4].flatten().tolist()}",
                      flush=True)
print("bad shapes:", bad)
