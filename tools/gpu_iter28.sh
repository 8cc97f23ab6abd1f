#!/bin/bash
# gat_ring staged grab metadata A/B (same box, back to back, twice)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gat.py tests/test_gpu_parity.py -x -q -m gpu -k "gat or narrow" > gpurun_out/it28_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it28_pytest.log
for r in 1 2; do for v in 0 1; do
  ATLAS_GAT_STAGED=$v timeout 900 python bench.py --workload igb-medium-gat --steps 5 --warmup 3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it28_gat_${v}_$r.json 2> gpurun_out/it28_gat_${v}_$r.err
done; done
