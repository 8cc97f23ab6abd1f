#!/bin/bash
# parity suite + smoke + bench (stable and tcgen05 transform backends)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_stable.json 2> gpurun_out/bench_stable.err
timeout 600 python bench.py --backend tcgen05 --no-cpu-baseline > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err
