#!/bin/bash
mkdir -p gpurun_out
for st in 0 19; do timeout 600 python tools/e2e_pipeline_probe.py 2 $st > gpurun_out/it12_e2e_pipe_st$st.txt 2>&1; done
timeout 900 python bench.py --no-cpu-baseline --no-cfg3 --no-alt > gpurun_out/it12_bench.json 2> gpurun_out/it12_bench.err
ATLAS_SWEEP_PROFILE=1 timeout 600 python tools/replay_probe.py 2400000 26 100 0.1 > gpurun_out/it12_probe_cfg2.txt 2>&1
