#!/bin/bash
# One gpurun pass producing a round's evidence: the default bench line, the
# GPU suite, launch lists and --set full captures of the heaviest relaxation
# launch of the headline (U-Net c=8) and of the north-star graph (C5 p=0.2).
#   TAG=r02 bash tools/gpu_round.sh
set -u
TAG=${TAG:-r02}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
bash tools/ncu_heaviest.sh k_relax_tile unet8_$TAG --workload unet --skip-len 8
bash tools/ncu_heaviest.sh k_relax_tile3 c5p02_$TAG --workload c5 --edge-prob 0.2
ls -la gpurun_out | tail -20
