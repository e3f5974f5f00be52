#!/bin/bash
# batching threshold of small levels into the persistent kernel (REMAT_SLT tests, REMAT_SLP preds)
cd $GRAFT_REPO_ROOT
source <(sed -n '/^probe()/,/^}/p' tools/knob_sweep.sh)
for c in "4194304 32768" "1048576 32768" "2097152 32768" "8388608 32768" "16777216 65536" "4194304 8192"; do
  set -- $c; echo "== SLT=$1 SLP=$2"; REMAT_SLT=$1 REMAT_SLP=$2 probe; REMAT_SLT=$1 REMAT_SLP=$2 timeout 300 python tools/configs_probe.py --no-cpu 2>/dev/null | grep -E "C1|C2"
done
