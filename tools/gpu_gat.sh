#!/bin/bash
# GAT + wide-row parity, IGB-Medium-shaped benches (GAT / SAGE / GCN)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gat.py -x -q > gpurun_out/pytest_gat.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gat.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload igb-medium-gat --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_igb_gat.json 2> gpurun_out/bench_igb_gat.err
timeout 900 python bench.py --workload igb-medium-gcn --steps 3 --warmup 3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/bench_igb_gcn.json 2> gpurun_out/bench_igb_gcn.err
timeout 600 python bench.py --no-cpu-baseline --no-alt > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
