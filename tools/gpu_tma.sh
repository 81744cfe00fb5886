#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
tail -2 gpurun_out/smoke.txt
if grep -q "smoke ok" gpurun_out/smoke.txt; then
  timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
  CHEBFD_TMA=0 timeout 600 python -m pytest tests -x -q -m gpu -k "spmmv or cheb_init or cfg1 or topi4" > gpurun_out/pytest_gpu_notma.txt 2>&1; tail -1 gpurun_out/pytest_gpu_notma.txt
  timeout 600 python tools/exp_locality.py "{\"CHEBFD_TMA_CFG\": \"0\"}" "{\"CHEBFD_TMA_CFG\": \"1\"}" "{\"CHEBFD_TMA\": \"0\"}" > gpurun_out/exp_loc.txt 2>&1; cut -c1-100 gpurun_out/exp_loc.txt
fi
