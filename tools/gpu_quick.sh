#!/bin/bash
# Quick GPU round trip: GPU tests (optionally filtered) + a short bench.
# Usage: bash tools/gpu_quick.sh [pytest -k expression]
mkdir -p gpurun_out
K=${1:-}
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q --timeout=600 -p no:cacheprovider -k "$K" > gpurun_out/pytest_gpu.log 2>&1
else
  timeout 1200 python -m pytest tests -m gpu -q --timeout=600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
fi
echo "pytest exit $?"; tail -25 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1
echo "bench exit $?"; tail -1 gpurun_out/bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('ms/step', round(d['ms_per_step'],3), 'GVU/s', round(d['value'],1), 'iters/s', round(d['admm_iters_per_s'],1), 'e2e', round(d['e2e']['value'],1))
print('roofline', r['kernel'], round(r['achieved'],1), round(r['frac'],3), r['components_ms'])"
