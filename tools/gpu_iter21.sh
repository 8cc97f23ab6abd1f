#!/bin/bash
# agg_tf_multi A/B: tests + cfg2 bench with the old and new narrow rings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "narrow or tolerance or transform_first" > gpurun_out/it21_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it21_pytest.log
for v in old new d8; do
  case $v in old) export ATLAS_TF_RING=old; unset ATLAS_TF_DEPTH;; new) unset ATLAS_TF_RING; unset ATLAS_TF_DEPTH;; d8) unset ATLAS_TF_RING; export ATLAS_TF_DEPTH=8;; esac
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cfg3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it21_cfg2_$v.json 2> gpurun_out/it21_cfg2_$v.err
done
unset ATLAS_TF_RING ATLAS_TF_DEPTH
timeout 600 ncu --kernel-name regex:agg_tf --set full --clock-control none --import-source on -c 1 -o gpurun_out/it21_tf python bench.py --steps 1 --warmup 3 --no-cfg3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it21_ncu.log 2>&1
