#!/bin/bash
# native CSC build (atomic scatter + segment sort) vs the radix-sort build
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -x -q -m gpu ) > gpurun_out/it43_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it43_pytest.log
for v in 1 0; do
  ATLAS_CSC_CUB=$v timeout 600 python tools/e2e_probe.py > gpurun_out/it43_e2e_cub$v.txt 2>&1
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cfg3 --no-alt --no-cpu-baseline > gpurun_out/it43_cfg2.json 2> gpurun_out/it43_cfg2.err
ATLAS_CSC_CUB=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cfg3 --no-alt --no-cpu-baseline > gpurun_out/it43_cfg2_cub.json 2> gpurun_out/it43_cfg2_cub.err
