#!/bin/bash
# GAT pass A with er fused into the epilogue (n = 128 kernels), A/B vs W_ext
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gat.py tests/test_gpu_multirank.py -x -q -m gpu > gpurun_out/it29_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it29_pytest.log
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -m gpu -k "gat or GAT" > gpurun_out/it29_scale.log 2>&1; echo "rc=$?" >> gpurun_out/it29_scale.log
for r in 1 2; do for v in 0 1; do
  ATLAS_GAT_ER=$v timeout 900 python bench.py --workload igb-medium-gat --steps 5 --warmup 3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it29_gat_${v}_$r.json 2> gpurun_out/it29_gat_${v}_$r.err
done; done
