#!/bin/bash
# Round-2 first pass: driver checks + launch list of the default bench.
bash tools/gpu_driver_check.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
ls -la gpurun_out
