# C4 view batch: ms/view and an ncu launch list of one 64-view batch (per-kernel totals)
python tools/views_time.py
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/views_launches.csv python tools/views_time.py > /dev/null 2>&1
python - <<'PY'
import csv, re, collections
rows = list(csv.reader(open('gpurun_out/views_launches.csv')))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; ki, vi = h.index('Kernel Name'), h.index('Metric Value')
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[hi + 1:]:
    n = re.sub(r'\(.*', '', r[ki]).replace('void ', '')
    tot[n] += float(r[vi].replace(',', '')) / 1e3; cnt[n] += 1
# 7 runs of 64 views: per view
for n, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{n:60s} {v / (7 * 64):8.1f} us/view  ({cnt[n]} launches)")
PY
