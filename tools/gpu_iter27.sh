#!/bin/bash
# L2 prefetch ahead of the transform producers' TMA loads
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "tcgen05 or transform" > gpurun_out/it27_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it27_pytest.log
for a in 0 8 16; do
  ATLAS_TF_L2AHEAD=$a timeout 600 python tools/transform_probe.py 2400000 > gpurun_out/it27_probe_$a.txt 2>&1
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cfg3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it27_cfg2.json 2> gpurun_out/it27_cfg2.err
