#!/bin/bash
# A/B of library variants (paper_1905_11722_b200/libremat_b200*.so) on the bench workloads
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do
for lib in paper_1905_11722_b200/libremat_b200*.so; do
  echo "== $lib"
  REMAT_B200_LIB=$PWD/$lib timeout 300 python tools/relax_probe.py $BIG; REMAT_B200_LIB=$PWD/$lib timeout 300 python tools/enum_probe.py; REMAT_B200_LIB=$PWD/$lib timeout 300 python tools/configs_probe.py --no-cpu
done
done > gpurun_out/ab_probe.log 2> gpurun_out/ab_probe.err
cat gpurun_out/ab_probe.log; tail -3 gpurun_out/ab_probe.err
