#!/bin/bash
# agg_tf_multi with staged grab metadata (shape A/B) + sweep pop marks
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py -x -q -m gpu -k "narrow or tolerance or transform_first or sweep" > gpurun_out/it22_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it22_pytest.log
for v in old 4 16 2; do
  if [ $v = old ]; then export ATLAS_TF_RING=old; unset ATLAS_TF_DEPTH; else unset ATLAS_TF_RING; export ATLAS_TF_DEPTH=$v; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cfg3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it22_cfg2_$v.json 2> gpurun_out/it22_cfg2_$v.err
done
unset ATLAS_TF_RING ATLAS_TF_DEPTH
ATLAS_SWEEP_PROFILE=1 timeout 900 python tools/replay_probe.py 2400000 26 100 0.1 > gpurun_out/it22_replay.txt 2>&1
