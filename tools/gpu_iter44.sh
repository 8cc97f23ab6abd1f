#!/bin/bash
mkdir -p gpurun_out
for v in 1 0; do
ATLAS_CSC_CUB=$v timeout 600 ncu --metrics gpu__time_duration.sum -k regex:"csc_|Onesweep|Upsweep|gather_u32|make_pairs|expand_sources|DeviceScan|RadixSort" -c 40 python tools/e2e_probe.py > gpurun_out/it44_ncu_cub$v.txt 2>&1
done
