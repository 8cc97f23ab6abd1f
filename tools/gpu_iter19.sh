#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_parity.py -x -q -m gpu -k "sweep or fast_path_metrics" > gpurun_out/it19_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it19_pytest.log
ATLAS_SWEEP_PROFILE=1 timeout 600 python tools/replay_probe.py 2400000 26 100 0.1 > gpurun_out/it19_probe_cfg2.txt 2>&1
ATLAS_SWEEP_PROFILE=1 timeout 600 python tools/replay_probe.py 2000000 12 128 0.1 > gpurun_out/it19_probe_u12.txt 2>&1
ATLAS_SWEEP_PROFILE=1 timeout 900 python bench.py --workload igb-large-sage-rank0of8-evict --steps 2 --warmup 1 > gpurun_out/it19_igb_evict.json 2> gpurun_out/it19_igb_evict.err
