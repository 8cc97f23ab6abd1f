#!/bin/bash
# round-2 refresh of every bench workload on HEAD
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/it33_cfg2.json 2> gpurun_out/it33_cfg2.err
for w in igb-medium-gcn igb-medium-sage; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it33_$w.json 2> gpurun_out/it33_$w.err
done
for w in papers100m-sage-rank0of8 igb-large-sage-rank0of8 igb-large-sage-rank0of8-evict; do
  timeout 1200 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/it33_$w.json 2> gpurun_out/it33_$w.err
done
