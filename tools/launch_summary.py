"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel time per
frame (median over the frames after the first; frames split on K1a)."""
import csv
import re
import statistics
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
frames, cur = [], []
for r in rows[hi + 1:]:
    name = re.sub(r"\(.*", "", r[ki].replace("(anonymous namespace)::", "").replace("unnamed>::", ""))
    if ("k_preprocess" in name or "k_geometry" in name) and cur:
        frames.append(cur)
        cur = []
    cur.append((name[-50:], float(r[vi].replace(",", ""))))
frames.append(cur)
use = frames[1:] if len(frames) > 1 else frames
per = {}
for f in use:
    agg = {}
    for n, v in f:
        agg[n] = agg.get(n, 0) + v
    for n, v in agg.items():
        per.setdefault(n, []).append(v)
med = {n: statistics.median(v) for n, v in per.items()}
tot = sum(med.values())
for n, v in sorted(med.items(), key=lambda x: -x[1]):
    print(f"{v / 1000:9.1f} us {100 * v / tot:5.1f}%  {n}")
print(f"total {tot / 1000:.1f} us per frame (median of {len(use)} frames)")
