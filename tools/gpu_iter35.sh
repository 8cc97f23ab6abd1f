#!/bin/bash
# f16 K=1024 N=256 pass A (IGB-Medium SAGE transform-first): 256-row tiles with one accumulator pair vs 128-row tiles
mkdir -p gpurun_out
for r in 1 2; do for v in 1 2; do
  ATLAS_TRANSFORM_H_SUB=$v timeout 900 python bench.py --workload igb-medium-sage --steps 3 --warmup 3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it35_sage_sub${v}_$r.json 2> gpurun_out/it35_sage_sub${v}_$r.err
done; done
