#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"sweep_kernel" --launch-count 1 -o /tmp/sw5 python tools/replay_probe.py 2400000 26 100 0.1 > gpurun_out/it18_ncu_sw.log 2>&1
ncu -i /tmp/sw5.ncu-rep --page details --csv > gpurun_out/it18_sw_details.csv 2>/dev/null
ncu -i /tmp/sw5.ncu-rep --page source --csv --print-source sass > gpurun_out/it18_sw_source.csv 2>/dev/null
ncu -i /tmp/sw5.ncu-rep --page raw --csv > gpurun_out/it18_sw_raw.csv 2>/dev/null
