#!/bin/bash
# One GPU session (single GPU): tests, smoke, bench, drop-in KATs, ncu of the
# apply_filter degree-step kernels.  Every step bounded by its own timeout.
# Usage: tools/gpu_session.sh [tag] [steps...]   steps: test smoke bench kat ncu_filter ncu_launch
cd "$(dirname "$0")/.."
tag=${1:-s}; shift
steps=${@:-test smoke bench kat ncu_filter}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used,memory.total --format=csv > gpurun_out/nvsmi_$tag.txt 2>&1
free -g >> gpurun_out/nvsmi_$tag.txt; nproc >> gpurun_out/nvsmi_$tag.txt
for s in $steps; do
case $s in
test) timeout 1500 python -m pytest tests -x -q -m gpu --durations=25 > gpurun_out/pytest_$tag.txt 2>&1
      echo "pytest rc=$?" >> gpurun_out/pytest_$tag.txt; tail -3 gpurun_out/pytest_$tag.txt ;;
smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.txt 2>&1
      echo "smoke rc=$?" >> gpurun_out/smoke_$tag.txt; tail -2 gpurun_out/smoke_$tag.txt ;;
bench) timeout 900 python bench.py --steps 50 --warmup 5 --e2e-steps 1 --cpu-steps 1 > gpurun_out/bench_$tag.txt 2>&1
      echo "bench rc=$?" >> gpurun_out/bench_$tag.txt; tail -c 600 gpurun_out/bench_$tag.txt ;;
kat) g++ -std=c++20 -O2 -Iinclude tests/cpp/kat_main.cpp -Lpaper_1803_02156_b200 -lchebfd_b200 \
        -Wl,-rpath,$PWD/paper_1803_02156_b200 -o /tmp/kat_main && timeout 300 /tmp/kat_main > gpurun_out/kat_$tag.txt 2>&1
      echo "kat rc=$?" >> gpurun_out/kat_$tag.txt; tail -6 gpurun_out/kat_$tag.txt ;;
ncu_filter) timeout 900 ncu --set full --clock-control none --import-source on -k regex:sell_b4_staged_kernel -s 14 -c 3 \
        -o gpurun_out/prof_filter_$tag -f python tools/prof_filter.py > gpurun_out/ncu_filter_$tag.txt 2>&1
      echo "ncu filter rc=$?" ;;
ncu_launch) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
        python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$tag.txt 2>&1
      echo "ncu launch rc=$?" ;;
ncu_cheb) timeout 900 ncu --set full --clock-control none --import-source on -k regex:sell_b4_ -s 5 -c 1 \
        -o gpurun_out/prof_cheb_$tag -f python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cheb_$tag.txt 2>&1
      echo "ncu cheb rc=$?" ;;
modes) timeout 600 python tools/step_modes.py > gpurun_out/modes_$tag.txt 2>&1; echo "modes rc=$?"; tail -2 gpurun_out/modes_$tag.txt ;;
modes_ab) timeout 900 python tools/step_modes.py --ab ${AB:-wpf=18,19,20,0} > gpurun_out/modes_ab_$tag.txt 2>&1; echo "modes ab rc=$?"; tail -2 gpurun_out/modes_ab_$tag.txt ;;
quick) timeout 900 python -m pytest tests -x -q -m gpu -k "parity or bloch or dist_peer or solve or dropin" > gpurun_out/pytest_$tag.txt 2>&1
      echo "pytest rc=$?" >> gpurun_out/pytest_$tag.txt; tail -3 gpurun_out/pytest_$tag.txt ;;
ksel) timeout 1500 python -m pytest tests -x -q -m gpu -k "$K" --durations=10 > gpurun_out/pytest_$tag.txt 2>&1
      echo "pytest rc=$?" >> gpurun_out/pytest_$tag.txt; tail -3 gpurun_out/pytest_$tag.txt ;;
tool) for t in $T; do timeout 1200 python tools/$t.py > gpurun_out/tool_${t}_$tag.txt 2>&1; echo "tool $t rc=$?"; \
      tail -c 1500 gpurun_out/tool_${t}_$tag.txt; done ;;
sanitize) for tl in memcheck racecheck synccheck; do timeout 900 compute-sanitizer --tool $tl --print-limit 20 \
      python tools/sanitize_cases.py > gpurun_out/sanitize_${tl}_$tag.txt 2>&1; echo "sanitize $tl rc=$?"; \
      tail -3 gpurun_out/sanitize_${tl}_$tag.txt; done ;;
esac
done
