"""Per-NVTX-phase kernel time from an `ncu --nvtx --metrics gpu__time_duration.sum --csv` log:
python tools/nvtx_summary.py gpurun_out/nvtx_phases.csv"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ni = [i for i, x in enumerate(h) if "Push/Pop_Range" in x][0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
per = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    ranges = re.findall(r":(tq:[a-z_]+):", r[ni])
    phase = ranges[-1] if ranges else "(none)"
    per[phase][r[ki].split("(")[0][-40:]].append(float(r[vi]) / 1e3)
for phase, ks in per.items():
    tot = sum(sum(v) for v in ks.values())
    print(f"{phase}: {tot:9.1f} us")
    for k, v in sorted(ks.items(), key=lambda x: -sum(x[1])):
        print(f"    {k:42s} n={len(v):3d} mean_us={sum(v) / len(v):8.2f}")
