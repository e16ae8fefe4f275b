#!/usr/bin/env python3
"""Top SASS instructions by warp-stall samples from `ncu --page source --print-source sass --csv`.

  python profiles/hot_sass.py <sass.csv> [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
ai, si, wi, ei = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
    h.index("Instructions Executed")
data = []
for r in rows[2:]:
    if len(r) <= max(wi, ei):
        continue
    try:
        data.append((int(r[wi] or 0), int(r[ei] or 0), r[ai], r[si]))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
print(f"total stall samples {tot}, instructions {sum(d[1] for d in data)}")
for w, e, a, s in sorted(data, reverse=True)[:top]:
    print(f"{w / tot:6.1%} {e:9d}  {a}  {s[:90]}")
