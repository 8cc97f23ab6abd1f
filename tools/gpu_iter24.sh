#!/bin/bash
# transform kernels under ncu (source-level stalls): cfg2 layer 0 f32 register split, cfg3 pass A f16
mkdir -p gpurun_out
timeout 900 ncu --kernel-name regex:transform_r_kernel --set full --clock-control none --import-source on -c 1 -o gpurun_out/it24_tr python bench.py --steps 1 --warmup 3 --no-cfg3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it24_ncu_tr.log 2>&1
timeout 900 ncu --kernel-name regex:transform_h_kernel --set full --clock-control none --import-source on -c 1 -o gpurun_out/it24_th python bench.py --workload igb-medium-gat --steps 1 --warmup 3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it24_ncu_th.log 2>&1
