#!/bin/bash
# memcheck / synccheck over the whole probe, racecheck on a reduced probe
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck; do
  ( time timeout 1500 $CS --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_probe.py ) > gpurun_out/sanitize_$tool.txt 2>&1
  echo "exit=$?" >> gpurun_out/sanitize_$tool.txt
done
( time SANITIZE_QUICK=1 timeout 2400 $CS --tool racecheck --print-limit 50 --error-exitcode 9 python tools/sanitize_probe.py ) > gpurun_out/sanitize_racecheck.txt 2>&1
echo "exit=$?" >> gpurun_out/sanitize_racecheck.txt
