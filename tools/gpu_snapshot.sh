#!/bin/bash
# Full evidence pass on one GPU: parity tests, smoke, bench lines (headline
# with cpu_baseline, C5, reference arm), ncu launch lists, relax DRAM traffic,
# one full capture of the relax kernel.  Everything lands in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --workload random-dag --edge-prob 0.3 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
bash tools/gpu_launches.sh
bash tools/gpu_traffic.sh unet
bash tools/gpu_prof.sh k_relax_tile 14
tail -n 2 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; head -c 600 gpurun_out/bench.json; echo
