#!/bin/bash
# streamed-W register split for 128 < N <= 192
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "3xtf32 or tolerance" > gpurun_out/it34_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it34_pytest.log
ATLAS_TRANSFORM_RS_WIDE=0 timeout 600 python tools/wide_probe.py > gpurun_out/it34_wide_off.txt 2>&1
timeout 600 python tools/wide_probe.py > gpurun_out/it34_wide_on.txt 2>&1
timeout 900 ncu --kernel-name regex:sweep_kernel --set full --clock-control none --import-source on -c 1 -o gpurun_out/it34_sweep python tools/replay_probe.py 2400000 26 100 0.1 > gpurun_out/it34_ncu_sweep.log 2>&1
