#!/bin/bash
# One GPU session: tests, smoke, short bench, launch list.  Every step bounded by timeout.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 600 python bench.py --steps 100 --warmup 5 --e2e-steps 1 --cpu-steps 1 > gpurun_out/bench.txt 2>&1
echo "bench rc=$?" >> gpurun_out/bench.txt
tail -3 gpurun_out/pytest_gpu.txt; tail -2 gpurun_out/smoke.txt; tail -3 gpurun_out/bench.txt
