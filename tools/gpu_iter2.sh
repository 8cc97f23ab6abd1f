#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_bounded.py tests/test_gpu_parity.py -x -q -m gpu -k "sweep or fast_path_metrics or bounded" > gpurun_out/it2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it2_pytest.log
timeout 300 python tools/transform_probe.py > gpurun_out/it2_transform_probe.txt 2>&1
ATLAS_SWEEP_PROFILE=1 timeout 600 python tools/replay_probe.py 2400000 26 100 0.1 > gpurun_out/it2_probe_cfg2.txt 2>&1
ATLAS_SWEEP_PROFILE=1 timeout 900 python bench.py --workload igb-large-sage-rank0of8-evict --steps 2 --warmup 1 > gpurun_out/it2_igb_evict.json 2> gpurun_out/it2_igb_evict.err
X=$(python -c "import torch;print(1)")
timeout 600 ncu --set full --clock-control none -k regex:"transform_t_kernel|transform_tc_kernel" -c 4 -o /tmp/tr python tools/transform_probe.py 300000 > gpurun_out/it2_ncu_tr.log 2>&1
ncu -i /tmp/tr.ncu-rep --page raw --csv > gpurun_out/it2_ncu_tr_raw.csv 2>/dev/null
ncu -i /tmp/tr.ncu-rep --page details --csv > gpurun_out/it2_ncu_tr_details.csv 2>/dev/null
