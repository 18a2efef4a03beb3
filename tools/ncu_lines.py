"""Aggregate an ncu source page (--print-source cuda,sass CSV) per CUDA source line."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = defaultdict(lambda: [0.0, 0.0, ""])
cur_file, hdr, line, src = "", None, None, ""
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8:
        continue
    if r[0]:
        line, src = r[0], r[1]
    ie = hdr.index("Instructions Executed")
    ws = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        a = agg[(cur_file, line)]
        a[0] += float(r[ie] or 0)
        a[1] += float(r[ws] or 0)
        a[2] = src
    except ValueError:
        pass
ti = sum(v[0] for v in agg.values()) or 1
tw = sum(v[1] for v in agg.values()) or 1
for (f, l), (i, w, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"inst {i / ti * 100:5.1f}%  stall {w / tw * 100:5.1f}%  {f}:{l:>4} {s.strip()[:90]}")
