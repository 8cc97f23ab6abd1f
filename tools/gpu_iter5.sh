#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_gds.py tests/test_disk_api.py tests/test_gpu_parity.py -x -q -m gpu -k "sweep or fast_path_metrics or gds or device_reader or disk or run_inference or run_layer" > gpurun_out/it5_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it5_pytest.log
cat > /tmp/tc24.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2605_09402_b200.engine import transform_typed
for k, n in ((64, 128), (100, 128), (128, 48)):
    x = torch.randn(2400000, k, device="cuda"); w = torch.randn(n, k, device="cuda") / k ** 0.5; b = torch.randn(n, device="cuda")
    for odt in (torch.float32, torch.float16):
        y = torch.empty(2400000, n, dtype=odt, device="cuda")
        os.environ["ATLAS_TRANSFORM_R"] = "0"; transform_typed(x, w, b, True, y, 1); torch.cuda.synchronize(); a = y.float().clone()
        os.environ.pop("ATLAS_TRANSFORM_R")
        for rep in range(3):
            transform_typed(x, w, b, True, y, 1); torch.cuda.synchronize()
            d = (y.float() - a).abs().max().item()
            print(k, n, odt, rep, d, flush=True)
PY
timeout 300 python /tmp/tc24.py > gpurun_out/it5_tc24.txt 2>&1
ATLAS_SWEEP_PROFILE=1 timeout 600 python tools/replay_probe.py 2400000 26 100 0.1 > gpurun_out/it5_probe_cfg2.txt 2>&1
ATLAS_SWEEP_PROFILE=1 timeout 900 python bench.py --workload igb-large-sage-rank0of8-evict --steps 2 --warmup 1 > gpurun_out/it5_igb_evict.json 2> gpurun_out/it5_igb_evict.err
timeout 900 python tools/io_bench.py > gpurun_out/it5_io_bench.json 2> gpurun_out/it5_io_bench.err
