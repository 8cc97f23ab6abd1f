#!/bin/bash
mkdir -p gpurun_out
ATLAS_SWEEP_PROFILE=1 timeout 600 python tools/replay_probe.py 2400000 26 100 0.1 > gpurun_out/it7_probe_cfg2.txt 2>&1
ATLAS_SWEEP_PROFILE=1 timeout 900 python bench.py --workload igb-large-sage-rank0of8-evict --steps 2 --warmup 1 > gpurun_out/it7_igb_evict.json 2> gpurun_out/it7_igb_evict.err
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/it7_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it7_pytest.log
timeout 600 python bench.py > gpurun_out/it7_bench.json 2> gpurun_out/it7_bench.err
ATLAS_BENCH_SHARE_GPU=1 ATLAS_BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/it7_bench_2rank.json 2> gpurun_out/it7_bench_2rank.err
timeout 900 python tools/io_bench.py > gpurun_out/it7_io_bench.json 2> gpurun_out/it7_io_bench.err
