#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tcgen05" > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
timeout 900 python bench.py --workload igb-medium-gcn --steps 3 --warmup 3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/bench_igb-medium-gcn.json 2> gpurun_out/bench_igb-medium-gcn.err
timeout 600 python bench.py --no-cpu-baseline --no-alt > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
