#!/bin/bash
# A/B of apply_filter's grouped X updates (3 / 2 / 1 degrees per X update): full-filter time and e2e (bench.py), one GPU.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "filter or host" > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -2 gpurun_out/pytest_gpu.txt
for v in "group3:CHEBFD_X_GROUP=3" "group2:CHEBFD_X_GROUP=2" "group1:CHEBFD_X_GROUP=1" "group3b:CHEBFD_X_GROUP=3"; do
  name=${v%%:*}; envs=${v#*:}
  ( [ -n "$envs" ] && export "$envs"
    timeout 600 python bench.py --steps 50 --warmup 5 --e2e-steps 1 --no-cpu-baseline --no-solve --no-panels 2>&1 | tail -1 ) > /tmp/f.txt
  python - "$name" /tmp/f.txt <<'PY' >> gpurun_out/filter_ab.txt
import json, sys
d = json.loads(open(sys.argv[2]).read())
print(f"{sys.argv[1]:10s} step {d['ms_per_step']:.3f} ms  chebfd_time {d['chebfd_time_s']:.3f} s  e2e {d['e2e']['value']:.0f} GF/s ({d['e2e']['seconds_per_call']:.3f} s)  mhz {d['clocks']['sm_mhz']}")
PY
done
cat gpurun_out/filter_ab.txt
