#!/bin/bash
# Round-end evidence: plain bench, launch list (warm, serialised), full captures of the two
# projector kernels (default cache control = flushed, as the recipe) under gpurun_out/TAG_*.
mkdir -p gpurun_out
TAG=$1
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5-geometry"
timeout 600 $CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 3000 --csv \
  --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "ncu launch exit $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"fp_persist_f32" -s 20 -c 1 -f -o gpurun_out/${TAG}_fp_full $CMD > gpurun_out/${TAG}_ncu_fp.log 2>&1
echo "ncu fp exit $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"bp_tile_kernel<float, \\(int\\)4>" -s 20 -c 1 -f -o gpurun_out/${TAG}_bp_full $CMD > gpurun_out/${TAG}_ncu_bp.log 2>&1
echo "ncu bp exit $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"fp_reduce_f32" -s 20 -c 1 -f -o gpurun_out/${TAG}_fpred_full $CMD > gpurun_out/${TAG}_ncu_fpred.log 2>&1
echo "ncu fp_reduce exit $?"
