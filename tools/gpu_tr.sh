#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "transform" > gpurun_out/pytest_tr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tr.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_stable3.json 2> gpurun_out/bench_stable3.err
timeout 600 python bench.py --backend tcgen05 --no-cpu-baseline > gpurun_out/bench_tc3.json 2> gpurun_out/bench_tc3.err
