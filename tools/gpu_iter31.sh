#!/bin/bash
# agg_sub_ring with staged grab metadata: A/B against the previous kernel on the papers100M rank slice
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "bit_exact or metrics" > gpurun_out/it31_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it31_pytest.log
for r in 1 2; do for v in old new; do
  if [ $v = old ]; then export ATLAS_LIB=libatlas_b200_old.so; else unset ATLAS_LIB; fi
  timeout 900 python bench.py --workload papers100m-sage-rank0of8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/it31_pap_${v}_$r.json 2> gpurun_out/it31_pap_${v}_$r.err
done; done
