#!/bin/bash
# ncu evidence for the dominant kernel: launch list + one full capture.  Single GPU.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.txt 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sell_b4_ -s 5 -c 1 \
  -o gpurun_out/prof_cheb python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
echo "full capture rc=$?"
# the degree steps of apply_filter: M_CHEB_NOX, M_CHEB_NOX, M_CHEB_X3 of the second call
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sell_b4_staged_kernel -s 14 -c 3 \
  -o gpurun_out/prof_filter python tools/prof_filter.py > gpurun_out/ncu_filter.txt 2>&1
echo "filter capture rc=$?"
