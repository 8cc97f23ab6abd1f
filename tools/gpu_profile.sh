#!/bin/bash
# Final-state profiles: launch list of the default bench command and full
# ncu captures of each workload's aggregation / transform kernels
# (exported to CSV on the box; the .ncu-rep files stay there).
mkdir -p gpurun_out /tmp/prof
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /tmp/prof/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"agg_ring|agg_tf_multi|transform_r_kernel" -c 5 -o /tmp/prof/cfg2_full python bench.py --steps 1 --warmup 0 --no-e2e --no-alt --no-cpu-baseline --no-cfg3 > /tmp/prof/ncu_cfg2.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"agg_ring|transform_h|agg_tf_multi" -c 5 -o /tmp/prof/igbgcn_full python bench.py --workload igb-medium-gcn --steps 1 --warmup 0 --no-e2e --no-alt --no-cpu-baseline > /tmp/prof/ncu_igbgcn.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"gat_ring|gat_bulk|transform_h" -c 4 -o /tmp/prof/igbgat_full python bench.py --workload igb-medium-gat --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /tmp/prof/ncu_igbgat.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"agg_sub_ring|transform_r_kernel|transform_tc" -c 4 -o /tmp/prof/papers_full python bench.py --workload papers100m-sage-rank0of8 --steps 1 --warmup 0 > /tmp/prof/ncu_papers.log 2>&1
for r in cfg2 igbgcn igbgat papers; do
  ncu -i /tmp/prof/${r}_full.ncu-rep --page raw --csv > gpurun_out/ncu_${r}_raw.csv 2>/dev/null
done
tail -3 /tmp/prof/*.log > gpurun_out/prof_logs.txt
ls -la gpurun_out
