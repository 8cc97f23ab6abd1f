#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "two_byte" > gpurun_out/it40_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it40_pytest.log
