#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gat_bulk|transform_h" -c 2 -o gpurun_out/gat2_full python bench.py --workload igb-medium-gat --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gat2.log 2>&1
