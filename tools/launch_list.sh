#!/bin/bash
# ncu launch list (gpu__time_duration per launch, no clock control) of a short bench run,
# summarised per kernel: bash tools/launch_list.sh TAG
mkdir -p gpurun_out
TAG=${1:-ll}
CMD="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c5-geometry"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv \
  --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu.log 2>&1
python - "$TAG" <<'PY'
import csv, sys, collections
tag = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/{tag}_launches.csv")) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki].split("(")[0][-40:]].append(float(r[vi]) / 1e3)
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{k:42s} n={len(v):4d} mean_us={sum(v)/len(v):8.2f} share={sum(v)/tot*100:5.1f}%")
PY
