#!/bin/bash
mkdir -p gpurun_out
free -g > gpurun_out/free.txt; nproc >> gpurun_out/free.txt
timeout 1500 python bench.py --workload igb-large-sage-rank0of8 --steps 3 --warmup 1 > gpurun_out/bench_large_slice.json 2> gpurun_out/bench_large_slice.err
