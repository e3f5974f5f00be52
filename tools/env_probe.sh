#!/bin/bash
# A/B of environment knobs (one process per setting): VAR and VALUES
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in $VALUES; do
  echo "== $VAR=$v"
  env $VAR=$v timeout 300 python tools/relax_probe.py $BIG
  env $VAR=$v timeout 300 python tools/enum_probe.py
  env $VAR=$v timeout 300 python tools/configs_probe.py --no-cpu
done > gpurun_out/env_probe.log 2> gpurun_out/env_probe.err
cat gpurun_out/env_probe.log; tail -3 gpurun_out/env_probe.err
