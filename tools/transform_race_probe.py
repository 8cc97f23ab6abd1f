"""Register-split transform vs the shared-memory kernel at 2.4M rows,
repeated, per stage-count override (diagnosing a nondeterministic
mismatch at K = 64)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2605_09402_b200.engine import transform_typed
for k, n in ((32, 128), (64, 128), (64, 64), (96, 128), (128, 128)):
    x = torch.randn(2400000, k, device="cuda"); w = torch.randn(n, k, device="cuda") / k ** 0.5; b = torch.randn(n, device="cuda")
    y = torch.empty(2400000, n, device="cuda")
    os.environ["ATLAS_TRANSFORM_R"] = "0"; transform_typed(x, w, b, True, y, 1); torch.cuda.synchronize(); a = y.clone()
    os.environ.pop("ATLAS_TRANSFORM_R")
    for st in (None, "3", "4", "6"):
        if st: os.environ["ATLAS_TRANSFORM_STAGES"] = st
        else: os.environ.pop("ATLAS_TRANSFORM_STAGES", None)
        bad = 0
        for rep in range(4):
            transform_typed(x, w, b, True, y, 1); torch.cuda.synchronize()
            d = (y - a).abs().max().item()
            bad += d > 1e-5
        print(k, n, "stages", st, "bad reps", bad, flush=True)
    os.environ.pop("ATLAS_TRANSFORM_STAGES", None)
