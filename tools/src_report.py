"""Per-source-line stall samples / executed instructions from an
`ncu --page source --print-source cuda,sass --csv` export (tools/ncu_kernel.sh)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = next(r for r in rows if r and r[0] == "Line No")
si, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
cur, out = None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > ii and r[0] not in ("", "Line No", "Function Name") and r[2] == "-":
        out.append((cur, r[0], r[1].strip()[:90], int(r[si] or 0), int(r[ii] or 0)))
ts = sum(o[3] for o in out) or 1
ti = sum(o[4] for o in out) or 1
print(f"samples {ts}  warp instructions {ti / 1e6:.1f}M")
for o in sorted(out, key=lambda o: -o[3])[:top]:
    print(f"{o[0][:14]:14s}:{o[1]:>4s} {100 * o[3] / ts:5.1f}% {o[4] / 1e6:7.2f}M  {o[2]}")
