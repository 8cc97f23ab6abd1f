#!/bin/bash
mkdir -p gpurun_out /tmp/p
cat > /tmp/p/tr1.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2605_09402_b200.engine import transform_typed
x = torch.randn(2400000, 128, device="cuda"); w = torch.randn(128, 128, device="cuda") / 11; b = torch.randn(128, device="cuda")
y = torch.empty(2400000, 128, device="cuda")
for t in ("0", "1"):
    os.environ["ATLAS_TRANSFORM_T"] = t
    for _ in range(2): transform_typed(x, w, b, True, y, 1)
torch.cuda.synchronize()
PY
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"transform_t_kernel|transform_tc_kernel" --launch-skip 1 --launch-count 3 -o /tmp/p/tr python /tmp/p/tr1.py > gpurun_out/p2_ncu_tr.log 2>&1
ncu -i /tmp/p/tr.ncu-rep --page raw --csv > gpurun_out/p2_tr_raw.csv 2>/dev/null
ncu -i /tmp/p/tr.ncu-rep --page details --csv > gpurun_out/p2_tr_details.csv 2>/dev/null
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"sweep_kernel" --launch-count 1 -o /tmp/p/sw python tools/replay_probe.py 600000 26 100 0.1 > gpurun_out/p2_ncu_sw.log 2>&1
ncu -i /tmp/p/sw.ncu-rep --page raw --csv > gpurun_out/p2_sw_raw.csv 2>/dev/null
ncu -i /tmp/p/sw.ncu-rep --page details --csv > gpurun_out/p2_sw_details.csv 2>/dev/null
ncu -i /tmp/p/sw.ncu-rep --page source --csv --print-source sass > gpurun_out/p2_sw_source.csv 2>/dev/null
ncu -i /tmp/p/tr.ncu-rep --page source --csv --print-source sass > gpurun_out/p2_tr_source.csv 2>/dev/null
ls -la gpurun_out/p2_*
