#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "user_host or metrics" > gpurun_out/it39_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it39_pytest.log
