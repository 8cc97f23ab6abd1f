"""Transform probe for 128 < N <= 192 (the papers100M SAGE head, K = 256 ->
172, f16 output): device time per call; run once with
ATLAS_TRANSFORM_RS_WIDE=0 (transform_tc_kernel, W streamed with x hi/lo
in shared memory) and once with the default (streamed-W register split).
Usage: wide_probe.py [rows]"""

import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2605_09402_b200.engine import transform_typed  # noqa: E402

PEAK = 6553.9


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 13_875_000
    for k, n, odt in [(256, 172, torch.float16), (256, 172, torch.float32),
                      (128, 136, torch.float32)]:
        x = torch.randn(rows, k, device="cuda")
        w = torch.randn(n, k, device="cuda") / k ** 0.5
        b = torch.randn(n, device="cuda")
        y = torch.empty(rows, n, dtype=odt, device="cuda")
        for _ in range(3):
            transform_typed(x, w, b, True, y, 1)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(5):
            transform_typed(x, w, b, True, y, 1)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / 5
        byts = rows * (k * 4 + n * y.element_size())
        ref = (x[:4096].double() @ w.double().T + b.double()).clamp_min(0)
        err = (y[:4096].double() - ref).abs().max().item()
        print(f"k={k} n={n} out={odt}: {ms:.3f} ms {byts / ms / 1e6:.0f} GB/s "
              f"({byts / ms / 1e6 / PEAK:.2f}) maxerr={err:.2e}", flush=True)


if __name__ == "__main__":
    main()
