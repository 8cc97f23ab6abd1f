#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_probe.py);
# summaries land in gpurun_out/sanitize_*.txt
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  ( time timeout 1500 $CS --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_probe.py ) > gpurun_out/sanitize_$tool.txt 2>&1
  echo "exit=$?" >> gpurun_out/sanitize_$tool.txt
done
ATLAS_ENGINE_GRID_MIN=1 timeout 900 $CS --tool racecheck --print-limit 50 --error-exitcode 9 python tools/sanitize_probe.py > gpurun_out/sanitize_racecheck_gridjobs.txt 2>&1
echo "exit=$?" >> gpurun_out/sanitize_racecheck_gridjobs.txt
