#!/bin/bash
# ncu --set full (warm L2) of the first launch, after SKIP, of kernels whose demangled name
# matches REGEX in the short bench command.  Usage: bash tools/gpu_ncu_one.sh TAG SKIP REGEX
mkdir -p gpurun_out
TAG=$1; S=$2; K=$3
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5-geometry"
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on --kernel-name-base demangled \
  -k "regex:$K" -s $S -c 1 -f -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu full $K exit $?"
