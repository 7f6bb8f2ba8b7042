#!/bin/bash
# per-kernel durations of the K-means encode (tools/km_time.py) under ncu (launch list only)
mkdir -p gpurun_out
TAG=${1:-km}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:km_ -c 40 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python tools/km_time.py > gpurun_out/${TAG}_ncu.log 2>&1
python - "$TAG" <<'PY'
import csv, sys, collections
tag = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/{tag}_launches.csv")) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki].split("(")[0][-40:]].append(float(r[vi]) / 1e3)
for k, v in d.items():
    print(f"{k:42s} n={len(v):3d} mean_us={sum(v)/len(v):8.2f}")
PY
