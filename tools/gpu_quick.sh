#!/bin/bash
# Quick gpurun pass: GPU parity tests + the two bench lines.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json | head -c 1500; tail -5 gpurun_out/bench.err
timeout 300 python bench.py --workload random-dag --edge-prob 0.3 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; head -c 1500 gpurun_out/bench_c5.json; tail -5 gpurun_out/bench_c5.err
