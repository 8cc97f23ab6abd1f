#!/bin/bash
mkdir -p gpurun_out
( echo "== bounce (default), /tmp"; timeout 120 python tools/gds_probe.py 100000 64 /tmp; echo "rc=$?"
  echo "== ATLAS_GDS=1, /tmp"; ATLAS_GDS=1 timeout 120 python tools/gds_probe.py 100000 64 /tmp; echo "rc=$?"
  mkdir -p $GRAFT_REPO_ROOT/gpurun_out/gdsdir
  echo "== ATLAS_GDS=1, repo dir"; ATLAS_GDS=1 timeout 120 python tools/gds_probe.py 100000 64 $GRAFT_REPO_ROOT/gpurun_out/gdsdir; echo "rc=$?"
  rm -rf $GRAFT_REPO_ROOT/gpurun_out/gdsdir; df -T /tmp | tail -1; lsmod 2>/dev/null | grep -i nvidia_fs ) > gpurun_out/it6_gds_probe.txt 2>&1
timeout 300 python tools/transform_race_probe.py > gpurun_out/it6_race.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_gds.py tests/test_disk_api.py -x -q -m gpu > gpurun_out/it6_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it6_pytest.log
ATLAS_SWEEP_PROFILE=1 timeout 600 python tools/replay_probe.py 2400000 26 100 0.1 > gpurun_out/it6_probe_cfg2.txt 2>&1
ATLAS_SWEEP_PROFILE=1 timeout 900 python bench.py --workload igb-large-sage-rank0of8-evict --steps 2 --warmup 1 > gpurun_out/it6_igb_evict.json 2> gpurun_out/it6_igb_evict.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"sweep_kernel" --launch-count 1 -o /tmp/sw2 python tools/replay_probe.py 2000000 12 128 0.1 > gpurun_out/it6_ncu_sw.log 2>&1
ncu -i /tmp/sw2.ncu-rep --page source --csv --print-source sass > gpurun_out/it6_sw_source.csv 2>/dev/null
ncu -i /tmp/sw2.ncu-rep --page raw --csv > gpurun_out/it6_sw_raw.csv 2>/dev/null
