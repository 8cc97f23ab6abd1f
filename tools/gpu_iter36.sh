#!/bin/bash
# L2 fetch granularity A/B (cudaLimitMaxL2FetchGranularity) on cfg2 and the GAT config
mkdir -p gpurun_out
python -c "
import torch,ctypes
torch.cuda.init()
lib=ctypes.CDLL('libcudart.so') if False else None
" 2>/dev/null
for r in 1 2; do for v in 0 32 64 128; do
  if [ $v = 0 ]; then unset ATLAS_L2_FETCH; else export ATLAS_L2_FETCH=$v; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cfg3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it36_cfg2_${v}_$r.json 2> gpurun_out/it36_cfg2_${v}_$r.err
done; done
unset ATLAS_L2_FETCH
timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:"agg_ring|agg_tf_multi" -c 6 python bench.py --steps 1 --warmup 0 --no-cfg3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it36_ncu_default.txt 2>&1
ATLAS_L2_FETCH=32 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:"agg_ring|agg_tf_multi" -c 6 python bench.py --steps 1 --warmup 0 --no-cfg3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it36_ncu_32.txt 2>&1
