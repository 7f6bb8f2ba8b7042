#!/bin/bash
# launch list + ncu --set full WITHOUT cache flush (warm L2, as inside the graph) of kernel regexes.
# Usage: bash tools/gpu_ncu_warm.sh TAG SKIP regex1 [regex2 ...]
mkdir -p gpurun_out
TAG=$1; S=$2; shift 2
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5-geometry"
timeout 600 $CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 3000 --csv \
  --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "ncu launch exit $?"
for K in "$@"; do
  timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:$K -s $S -c 1 \
    -f -o gpurun_out/${TAG}_${K}_full $CMD > gpurun_out/${TAG}_ncu_${K}.log 2>&1
  echo "ncu full $K exit $?"
done
