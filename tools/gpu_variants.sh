#!/bin/bash
# Parity tests, then short kernel-only bench runs of the tuning variants given as
# "NAME:ENV=V,ENV2=V" arguments (default variant first).  Single GPU, bounded.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -2 gpurun_out/pytest_gpu.txt
: > gpurun_out/variants.txt
for v in "default:" "$@"; do
  name=${v%%:*}; envs=${v#*:}
  ( IFS=','; for e in $envs; do [ -n "$e" ] && export "$e"; done
    timeout 300 python bench.py --steps 150 --warmup 5 --no-e2e --no-cpu-baseline --no-solve 2>&1 | tail -1 ) > /tmp/v.txt
  python - "$name" /tmp/v.txt >> gpurun_out/variants.txt <<'PY'
import json, sys
name, f = sys.argv[1], sys.argv[2]
t = open(f).read().strip()
try:
    d = json.loads(t)
    print(f"{name:24s} ms/step {d['ms_per_step']:.4f}  frac {d['roofline']['frac']:.4f}  sm_mhz {d['clocks']['sm_mhz']} W {d['clocks'].get('power_w')} {d['clocks']['reasons']}")
except Exception:
    print(f"{name:24s} FAILED: {t[-300:]}")
PY
done
cat gpurun_out/variants.txt
