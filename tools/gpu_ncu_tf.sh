#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"agg_tf_ring|agg_ring" -c 3 -o gpurun_out/tf_full python bench.py --steps 1 --warmup 0 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/ncu_tf.log 2>&1
