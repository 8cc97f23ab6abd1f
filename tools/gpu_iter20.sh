#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "tcgen05 or transform" > gpurun_out/it20_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it20_pytest.log
timeout 300 python tools/transform_probe.py 2400000 3000000 > gpurun_out/it20_transform_probe.txt 2>&1
timeout 900 python bench.py --workload papers100m-sage-rank0of8 --steps 3 --warmup 3 > gpurun_out/it20_papers.json 2> gpurun_out/it20_papers.err
timeout 900 python bench.py --workload igb-medium-sage --steps 3 --warmup 3 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/it20_igbsage.json 2> gpurun_out/it20_igbsage.err
