#!/bin/bash
# packed 16-entry sweep windows A/B; user host backend test
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_bounded.py tests/test_gpu_parity.py -x -q -m gpu -k "sweep or bounded or metrics or user_host or bit_exact" > gpurun_out/it38_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it38_pytest.log
for v in 0 1; do
  ATLAS_SWEEP_PK=$v ATLAS_SWEEP_PROFILE=1 timeout 900 python tools/replay_probe.py 2400000 26 100 0.1 > gpurun_out/it38_replay_pk$v.txt 2>&1
done
for v in 0 1; do
  ATLAS_SWEEP_PK=$v timeout 1200 python bench.py --workload igb-large-sage-rank0of8-evict --steps 3 --warmup 3 > gpurun_out/it38_evict_pk$v.json 2> gpurun_out/it38_evict_pk$v.err
done
