#!/bin/bash
# agg_tf_multi with staged grab metadata (shape A/B) + sweep pop marks
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py -x -q -m gpu -k "narrow or tolerance or transform_first" > gpurun_out/it25_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it25_pytest.log
for v in 0 6 7 9 4; do
  if [ $v = old ]; then export ATLAS_TF_RING=old; unset ATLAS_TF_DEPTH; else unset ATLAS_TF_RING; export ATLAS_TF_DEPTH=$v; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cfg3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it25_cfg2_$v.json 2> gpurun_out/it25_cfg2_$v.err
done
unset ATLAS_TF_RING ATLAS_TF_DEPTH
timeout 900 ncu --kernel-name regex:transform_r_kernel --set full --clock-control none --import-source on -c 1 -o gpurun_out/it25_tr python bench.py --steps 1 --warmup 3 --no-cfg3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it25_ncu_tr.log 2>&1
timeout 900 ncu --kernel-name regex:transform_h_kernel --set full --clock-control none --import-source on -c 1 -o gpurun_out/it25_th python bench.py --workload igb-medium-gat --steps 1 --warmup 3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it25_ncu_th.log 2>&1
