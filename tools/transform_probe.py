"""Transform kernel probe: device time of the tcgen05 transform on
cfg2-sized shapes for each kernel variant: "smem" = x hi/lo in shared
memory stages (ATLAS_TRANSFORM_R=0), "tmemW" = W in TMEM with the
transposed product (ATLAS_TRANSFORM_T=1), "regsplit" = x split in registers
into TMEM A stages (the default), and output dtype.
Usage: transform_probe.py [rows]"""

import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2605_09402_b200.engine import transform_typed  # noqa: E402

PEAK = 6544.0


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 2_400_000
    for k, n in [(100, 128), (128, 128), (128, 48), (128, 64), (64, 128),
                 (256, 128)]:
        x = torch.randn(rows, k, device="cuda")
        w = torch.randn(n, k, device="cuda") / k ** 0.5
        b = torch.randn(n, device="cuda")
        for odt in (torch.float32, torch.float16):
            y = torch.empty(rows, n, dtype=odt, device="cuda")
            res = []
            for t, env in (("smem", {"ATLAS_TRANSFORM_R": "0"}),
                           ("tmemW", {"ATLAS_TRANSFORM_T": "1"}),
                           ("regsplit", {})):
                for key in ("ATLAS_TRANSFORM_R", "ATLAS_TRANSFORM_T"):
                    os.environ.pop(key, None)
                os.environ.update(env)
                for _ in range(3):
                    transform_typed(x, w, b, True, y, 1)
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                ev[0].record()
                for _ in range(10):
                    transform_typed(x, w, b, True, y, 1)
                ev[1].record()
                torch.cuda.synchronize()
                ms = ev[0].elapsed_time(ev[1]) / 10
                byts = rows * (k * 4 + n * y.element_size())
                res.append(f"{t} {ms:.3f} ms {byts / ms / 1e6:.0f} GB/s "
                           f"({byts / ms / 1e6 / PEAK:.2f})")
                if t == "smem":
                    y0 = y.float().clone()
                else:
                    res[-1] += f" d={(y.float() - y0).abs().max().item():.1e}"
            print(f"k={k} n={n} out={odt}: " + " | ".join(res), flush=True)


def f16_inputs(rows):
    """transform_h (f16 x, kind::f16): 128-row vs 256-row tiles."""
    for k, n in [(1024, 128), (1024, 19), (1024, 136)]:
        x = torch.randn(rows, k, device="cuda").half()
        w = torch.randn(n, k, device="cuda") / k ** 0.5
        b = torch.randn(n, device="cuda")
        y = torch.empty(rows, n, device="cuda")
        res = []
        for sub in ("1", "2") if n <= 128 else ("1", "2"):
            os.environ["ATLAS_TRANSFORM_H_SUB"] = sub
            for _ in range(3):
                transform_typed(x, w, b, True, y, 1)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            for _ in range(10):
                transform_typed(x, w, b, True, y, 1)
            ev[1].record()
            torch.cuda.synchronize()
            ms = ev[0].elapsed_time(ev[1]) / 10
            byts = rows * (k * 2 + n * 4)
            res.append(f"sub={sub} {ms:.3f} ms {byts / ms / 1e6:.0f} GB/s "
                       f"({byts / ms / 1e6 / PEAK:.2f})")
            if sub == "1":
                y1 = y.clone()
            else:
                res[-1] += f" d={(y - y1).abs().max().item():.1e}"
        os.environ.pop("ATLAS_TRANSFORM_H_SUB", None)
        print(f"f16 x k={k} n={n}: " + " | ".join(res), flush=True)


if __name__ == "__main__":
    main()
    f16_inputs(int(sys.argv[2]) if len(sys.argv) > 2 else 3_000_000)
