#!/bin/bash
# A/B of every library build paper_1905_11722_b200/libremat_b200*.so on
# tools/ab_relax.py cases ($CASES), two alternating rounds.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for r in 1 2; do
  for lib in paper_1905_11722_b200/libremat_b200*.so; do
    REMAT_B200_LIB=$PWD/$lib timeout 600 python tools/ab_relax.py $CASES
  done
done 2>&1 | tee gpurun_out/ab_libs.log
