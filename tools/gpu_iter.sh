#!/bin/bash
# iteration check: transform + sweep parity, replay phase profile, A/B benches
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py -x -q -m gpu -k "tcgen05 or transform or sweep or fast_path_metrics" > gpurun_out/iter_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/iter_pytest.log
ATLAS_SWEEP_PROFILE=1 timeout 600 python tools/replay_probe.py 2400000 26 100 0.1 > gpurun_out/iter_probe_cfg2.txt 2>&1
ATLAS_SWEEP_PROFILE=1 timeout 900 python bench.py --workload igb-large-sage-rank0of8-evict --steps 1 --warmup 1 > gpurun_out/iter_igb_evict.json 2> gpurun_out/iter_igb_evict.err
for t in 0 1; do
ATLAS_TRANSFORM_T=$t timeout 600 python bench.py --no-cfg3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/iter_cfg2_t$t.json 2> gpurun_out/iter_cfg2_t$t.err
done
