#!/bin/bash
mkdir -p gpurun_out
for w in igb-medium-gat igb-medium-gcn igb-medium-sage; do
timeout 900 python bench.py --workload $w --embed-dtype f16 --steps 3 --warmup 3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/bench_${w}_f16.json 2> gpurun_out/bench_${w}_f16.err
done
timeout 600 python bench.py --embed-dtype f16 --no-cpu-baseline --no-alt --no-e2e > gpurun_out/bench_cfg2_f16.json 2> gpurun_out/bench_cfg2_f16.err
