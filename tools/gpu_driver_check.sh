#!/bin/bash
# What the driver runs at round end: GPU tests, smoke, default bench,
# reference arm.
mkdir -p gpurun_out
( time timeout 1200 python -m pytest tests -x -q -m gpu ) > gpurun_out/drv_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/drv_pytest.log
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/drv_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/drv_smoke.log
( time timeout 900 python bench.py ) > gpurun_out/drv_bench.json 2> gpurun_out/drv_bench.err; echo "rc=$?" >> gpurun_out/drv_bench.err
( time timeout 900 python bench.py --impl reference ) > gpurun_out/drv_ref.json 2> gpurun_out/drv_ref.err; echo "rc=$?" >> gpurun_out/drv_ref.err
