"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel time of the last frame."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
frames, cur = [], []
for r in rows[hi + 1:]:
    name = re.sub(r"\(.*", "", r[ki])
    if ("k_preprocess" in name or "k_geometry" in name) and cur:
        frames.append(cur)
        cur = []
    cur.append((name[-50:], float(r[vi].replace(",", ""))))
frames.append(cur)
f = frames[-1]
tot = sum(v for _, v in f)
agg = {}
for n, v in f:
    agg[n] = agg.get(n, 0) + v
for n, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{v / 1000:9.1f} us {100 * v / tot:5.1f}%  {n}")
print(f"total {tot / 1000:.1f} us over {len(f)} launches")
