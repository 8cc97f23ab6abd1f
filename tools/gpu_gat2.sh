#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gat.py -x -q > gpurun_out/pytest_gat.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gat.log
timeout 900 python bench.py --workload igb-medium-gat --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_igb_gat.json 2> gpurun_out/bench_igb_gat.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gat_bulk|transform_tc" -c 2 -o gpurun_out/gat_full python bench.py --workload igb-medium-gat --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gat.log 2>&1
