#!/bin/bash
# ncu launch lists (gpu__time_duration per kernel) of one U-Net c=8 and one C5 p=0.3 solve
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_unet.csv python tools/solve_once.py > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python tools/solve_once.py --workload random-dag > /dev/null 2>&1
echo done
