#!/bin/bash
# round-2 end evidence on HEAD: driver checks, then profiles
bash tools/gpu_driver_check.sh
bash tools/gpu_profile.sh
