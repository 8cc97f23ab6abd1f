#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_bounded.py tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -m gpu -k "sweep or fast_path_metrics or bounded or tcgen05 or transform or cfg2_tcgen05" > gpurun_out/it3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it3_pytest.log
timeout 300 python tools/transform_probe.py > gpurun_out/it3_transform_probe.txt 2>&1
ATLAS_SWEEP_PROFILE=1 timeout 600 python tools/replay_probe.py 2400000 26 100 0.1 > gpurun_out/it3_probe_cfg2.txt 2>&1
ATLAS_SWEEP_PROFILE=1 timeout 900 python bench.py --workload igb-large-sage-rank0of8-evict --steps 2 --warmup 1 > gpurun_out/it3_igb_evict.json 2> gpurun_out/it3_igb_evict.err
timeout 600 python bench.py --no-cfg3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/it3_cfg2.json 2> gpurun_out/it3_cfg2.err
