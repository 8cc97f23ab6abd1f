#!/bin/bash
mkdir -p gpurun_out
ATLAS_BENCH_INFLIGHT=3 timeout 900 python bench.py --no-cpu-baseline --no-cfg3 --no-alt > gpurun_out/it13_bench_if3.json 2> gpurun_out/it13_bench_if3.err
bash tools/gpu_sanitize.sh
