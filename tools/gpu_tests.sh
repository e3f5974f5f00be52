#!/bin/bash
# gpurun: selected GPU tests (args) or the whole -m gpu suite, plus smoke().
mkdir -p gpurun_out
T=${1:-tests}
timeout 1500 python -m pytest $T -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
