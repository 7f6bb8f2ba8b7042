"""Top warp-stall reasons (pc sampling) of an ncu report: python tools/stalls.py rep.ncu-rep"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
for v in r[2:]:
    print(v[h.index("Kernel Name")][:80], v[h.index("gpu__time_duration.sum")], "us")
    it = []
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try: it.append((float(v[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError: pass
    tot = sum(x for x, _ in it) or 1
    print("   " + ", ".join(f"{k} {100*x/tot:.0f}%" for x, k in sorted(it, reverse=True)[:7]))
    for k in ["smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum"]:
        if k in h: print(f"   {k} = {v[h.index(k)]}")
