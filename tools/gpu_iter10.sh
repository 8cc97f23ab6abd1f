#!/bin/bash
mkdir -p gpurun_out
ATLAS_SWEEP_DIAG_NO_FAR=2 ATLAS_SWEEP_PROFILE=1 timeout 600 python tools/replay_probe.py 2000000 12 128 0.1 > gpurun_out/it10_probe_u12_noatomics.txt 2>&1
ATLAS_SWEEP_DIAG_NO_FAR=2 ATLAS_SWEEP_PROFILE=1 timeout 600 python tools/replay_probe.py 2400000 26 100 0.1 > gpurun_out/it10_probe_cfg2_noatomics.txt 2>&1
for n in 3 4; do ATLAS_BENCH_INFLIGHT=$n timeout 900 python bench.py --no-cpu-baseline --no-cfg3 --no-alt > gpurun_out/it10_bench_inflight$n.json 2> gpurun_out/it10_bench_inflight$n.err; done
