#!/bin/bash
# ncu full capture of one relaxation launch (args: kernel regex, skip count, extra solve args)
mkdir -p gpurun_out
K=${1:-k_relax_tile}; S=${2:-40}; shift 2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/prof -f python tools/solve_once.py "$@" > gpurun_out/ncu_prof.log 2>&1
tail -3 gpurun_out/ncu_prof.log
