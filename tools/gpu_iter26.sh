#!/bin/bash
# gat_ring with staged grab metadata; narrow transform-first shapes for 20-wide z (IGB-Medium GCN)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gat.py tests/test_gpu_parity.py -x -q -m gpu -k "gat or narrow or tolerance or transform_first" > gpurun_out/it26_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it26_pytest.log
timeout 900 python bench.py --workload igb-medium-gat --steps 5 --warmup 3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it26_gat.json 2> gpurun_out/it26_gat.err
for v in old 0 12 13; do
  if [ $v = old ]; then export ATLAS_TF_RING=old; unset ATLAS_TF_DEPTH; else unset ATLAS_TF_RING; export ATLAS_TF_DEPTH=$v; fi
  timeout 900 python bench.py --workload igb-medium-gcn --steps 3 --warmup 3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it26_gcn_$v.json 2> gpurun_out/it26_gcn_$v.err
done
