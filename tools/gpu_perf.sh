#!/bin/bash
# parity (all GPU tests) + every bench workload; results in gpurun_out/
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
for w in igb-medium-gat igb-medium-gcn igb-medium-sage; do
timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
for w in papers100m-sage-rank0of8 igb-large-sage-rank0of8; do
timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
