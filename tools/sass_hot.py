"""Instruction-count breakdown of one ncu --set full capture by straight-line SASS blocks
(consecutive instructions with equal execution counts):
python tools/sass_hot.py rep.ncu-rep [top]"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
isrc, ie, ist = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ie]) for r in data)
print(rows[0][1][:100], "| warp instr", tot)
blocks, cur = [], None
for i, r in enumerate(data):
    s, e, w = r[isrc].strip()[:50], int(r[ie]), int(r[ist])
    if cur and cur[2] == e:
        cur[1] += 1; cur[3] += w; cur[4].append(s)
    else:
        if cur: blocks.append(cur)
        cur = [i, 1, e, w, [s]]
blocks.append(cur)
for b in sorted(blocks, key=lambda b: -b[1] * b[2])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"@{b[0]:5d} n={b[1]:4d} exec={b[2]:9d} {100*b[1]*b[2]/tot:5.1f}% stall={b[3]:6d}  {b[4][0]} .. {b[4][-1]}")
