#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/it14_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it14_pytest.log
ATLAS_SWEEP_PROFILE=1 timeout 600 python tools/replay_probe.py 2400000 26 100 0.1 > gpurun_out/it14_probe_cfg2.txt 2>&1
ATLAS_SWEEP_PROFILE=1 timeout 600 python tools/replay_probe.py 2000000 12 128 0.1 > gpurun_out/it14_probe_u12.txt 2>&1
ATLAS_SWEEP_PROFILE=1 timeout 900 python bench.py --workload igb-large-sage-rank0of8-evict --steps 2 --warmup 1 > gpurun_out/it14_igb_evict.json 2> gpurun_out/it14_igb_evict.err
timeout 600 python tools/e2e_pipeline_probe.py 2 19 > gpurun_out/it14_e2e_pipe.txt 2>&1
timeout 900 python bench.py > gpurun_out/it14_bench.json 2> gpurun_out/it14_bench.err
timeout 300 python tools/transform_probe.py 2400000 3000000 > gpurun_out/it14_transform_probe.txt 2>&1
