#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/it16_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it16_pytest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/it16_bench.json 2> gpurun_out/it16_bench.err
