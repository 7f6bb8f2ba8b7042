#!/bin/bash
# One GPU round trip: the GPU test suite, smoke(), a short bench, the ncu launch list
# and one `ncu --set full` capture of each projector kernel.
# Usage (from the repo root, via gpurun): bash tools/gpu_check.sh [pytest-args]
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep -E "Model name|^CPU\(s\)"
timeout 1500 python -m pytest tests -m gpu -q --timeout=600 -p no:cacheprovider "$@" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?"
tail -40 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?"; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1
echo "bench exit $?"; tail -2 gpurun_out/bench.log | cut -c1-4000
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/bench_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu launch exit $?"
for K in bp_kernel fp_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 1 \
    -f -o gpurun_out/${K}_full $CMD > gpurun_out/ncu_${K}.log 2>&1
  echo "ncu full $K exit $?"
done
