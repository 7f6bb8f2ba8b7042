#!/bin/bash
# ncu --set full of the K-means kernels given as regexes (one launch each) in tools/km_time.py
mkdir -p gpurun_out
TAG=$1; shift
for K in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-2} -c 1 \
    -f -o gpurun_out/${TAG}_${K} python tools/km_time.py > gpurun_out/${TAG}_ncu_${K}.log 2>&1
  echo "ncu $K exit $?"
done
