#!/bin/bash
# sweep replay: parity (goldens through the sweep, A/B vs the per-element
# machine, ablation integers) and timing (cfg2 10 % slots, IGB-Large slice)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_parity.py tests/test_ablation.py -x -q -m gpu -k "sweep or fast_path_metrics or ablation or criteria" > gpurun_out/sweep_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sweep_pytest.log
timeout 600 python tools/replay_probe.py 2400000 26 100 0.1 > gpurun_out/sweep_probe_cfg2_10pct.txt 2>&1
ATLAS_SWEEP=0 timeout 600 python tools/replay_probe.py 2400000 26 100 0.1 > gpurun_out/sweep_probe_cfg2_10pct_old.txt 2>&1
timeout 900 python bench.py --workload igb-large-sage-rank0of8-evict --steps 2 --warmup 1 > gpurun_out/sweep_bench_igb_large_evict.json 2> gpurun_out/sweep_bench_igb_large_evict.err
