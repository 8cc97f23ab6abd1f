#!/bin/bash
# round-2 refresh: every bench workload + ncu launch list and full captures
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/f_bench_cfg2.json 2> gpurun_out/f_bench_cfg2.err
for w in igb-medium-gcn igb-medium-sage; do
timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/f_bench_$w.json 2> gpurun_out/f_bench_$w.err
done
for w in papers100m-sage-rank0of8 igb-large-sage-rank0of8; do
timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/f_bench_$w.json 2> gpurun_out/f_bench_$w.err
done
bash tools/gpu_profile.sh
