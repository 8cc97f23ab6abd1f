#!/bin/bash
# span order statistics by radix select (vs device sort), control plane queued first, agg_sub_ring staged metadata
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_gpu_bounded.py tests/test_disk_api.py -x -q -m gpu > gpurun_out/it32_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it32_pytest.log
for r in 1 2; do
  for v in sort sel first; do
    unset ATLAS_SPAN_SORT ATLAS_CTL_FIRST
    [ $v = sort ] && export ATLAS_SPAN_SORT=1
    [ $v = first ] && export ATLAS_CTL_FIRST=1
    timeout 600 python bench.py --steps 5 --warmup 3 --no-cfg3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it32_cfg2_${v}_$r.json 2> gpurun_out/it32_cfg2_${v}_$r.err
  done
done
unset ATLAS_SPAN_SORT ATLAS_CTL_FIRST
for v in old new; do
  if [ $v = old ]; then export ATLAS_LIB=libatlas_b200_old.so; else unset ATLAS_LIB; fi
  timeout 900 python bench.py --workload papers100m-sage-rank0of8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/it32_pap_${v}.json 2> gpurun_out/it32_pap_${v}.err
done
