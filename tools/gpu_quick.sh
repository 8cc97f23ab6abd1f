#!/bin/bash
# transform parity + bench + full ncu captures of agg_ring / stable transform
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "transform" > gpurun_out/pytest_tr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tr.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_stable2.json 2> gpurun_out/bench_stable2.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:agg_ring -c 1 -o gpurun_out/agg_ring_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_agg.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transform_stable_tiled -c 2 -o gpurun_out/tr_stable_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_tr.log 2>&1
ls -la gpurun_out
