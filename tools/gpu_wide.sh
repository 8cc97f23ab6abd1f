#!/bin/bash
# wide-row (1024-d f16) parity + IGB-Medium-shaped bench + ncu of agg_bulk
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload igb-medium-sage --steps 3 --warmup 3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/bench_igb_sage.json 2> gpurun_out/bench_igb_sage.err
timeout 900 python bench.py --workload igb-medium-gcn --steps 3 --warmup 3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/bench_igb_gcn.json 2> gpurun_out/bench_igb_gcn.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:agg_bulk -c 1 -o gpurun_out/agg_bulk_full python bench.py --workload igb-medium-gcn --steps 1 --warmup 0 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/ncu_bulk.log 2>&1
ls -la gpurun_out
