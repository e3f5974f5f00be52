#!/bin/bash
# env-knob combinations of the level planner (REMAT_WANT_MUL, REMAT_SPLIT_MUL)
cd $GRAFT_REPO_ROOT
source <(sed -n '/^probe()/,/^}/p' tools/knob_sweep.sh)
for c in "64 2" "32 4" "16 4" "32 6" "32 8" "16 8" "32 3"; do
  set -- $c; echo "== WANT_MUL=$1 SPLIT_MUL=$2"; REMAT_WANT_MUL=$1 REMAT_SPLIT_MUL=$2 probe
done
