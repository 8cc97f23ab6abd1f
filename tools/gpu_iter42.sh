#!/bin/bash
# sanitizers over every kernel family after the round-2b changes
mkdir -p gpurun_out
timeout 300 python tools/sanitize_probe.py > gpurun_out/it42_plain.txt 2>&1; echo "exit=$?" >> gpurun_out/it42_plain.txt
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  ( time timeout 1500 $CS --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_probe.py ) > gpurun_out/it42_sanitize_$tool.txt 2>&1
  echo "exit=$?" >> gpurun_out/it42_sanitize_$tool.txt
done
