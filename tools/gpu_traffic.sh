#!/bin/bash
# DRAM bytes + duration of every k_relax_tile launch of one bench-workload solve
# (ncu, cold-cache, serialised) -> gpurun_out/traffic_<workload>.csv
mkdir -p gpurun_out
W=${1:-unet}; shift
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:k_relax --csv --log-file gpurun_out/traffic_$W.csv python tools/solve_once.py --workload $W "$@" > /dev/null 2>&1
echo traffic done
