#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gds.py tests/test_gpu_parity.py tests/test_gpu_sweep.py -x -q -m gpu -k "gds or device_reader or f16_input or 3xtf32 or sweep or fast_path_metrics" > gpurun_out/it8_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it8_pytest.log
timeout 300 python tools/transform_probe.py 2400000 3000000 > gpurun_out/it8_transform_probe.txt 2>&1
ATLAS_SWEEP_PROFILE=1 timeout 600 python tools/replay_probe.py 2400000 26 100 0.1 > gpurun_out/it8_probe_cfg2.txt 2>&1
ATLAS_SWEEP_PROFILE=1 timeout 600 python tools/replay_probe.py 2000000 12 128 0.1 > gpurun_out/it8_probe_u12.txt 2>&1
ATLAS_SWEEP_DIAG_NO_FAR=1 ATLAS_SWEEP_PROFILE=1 timeout 600 python tools/replay_probe.py 2000000 12 128 0.1 > gpurun_out/it8_probe_u12_nofar.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/it8_bench.json 2> gpurun_out/it8_bench.err
timeout 900 python tools/io_bench.py > gpurun_out/it8_io_bench.json 2> gpurun_out/it8_io_bench.err
