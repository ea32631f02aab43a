"""Aggregates an ncu source export (tools/ncu_kernel.sh) of k_blend16 into
regions (sort / staging / transpose / walk / replay) by source line ranges."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
src = open(sys.argv[2] if len(sys.argv) > 2 else "paper_2603_18707_b200/csrc/blend.cu").read().splitlines()


def find(pat, start=0):
    for i in range(start, len(src)):
        if re.search(pat, src[i]):
            return i + 1
    raise KeyError(pat)


k = find(r"__global__ void __launch_bounds__\(128, .*\) k_blend16")
ranges = {
    "walk": (find(r"^struct Frag \{"), find(r"^// Exact replay of one flagged pixel")),
    "replay": (find(r"^// Exact replay of one flagged pixel"), find(r"^// CAPR: rounds")),
    "cover(row_pairs2)": (find(r"row_pairs2\(int row"), find(r"^// Record-local split")),
    "transpose": (find(r"warp_transpose32\(uint32_t x"), find(r"^// ---- packed fp32 pairs")),
    "blend16 prologue": (k, find(r"for \(int base = 0; base < L; base \+= kB16\)", k)),
    "batch barrier+stage": (find(r"for \(int base = 0; base < L; base \+= kB16\)", k), find(r"coverage of \{q <= q_hi\}", k)),
    "stage cover loop": (find(r"coverage of \{q <= q_hi\}", k), find(r"__syncthreads_or\(needs_clamp\)", k)),
    "barrier+prefetch": (find(r"__syncthreads_or\(needs_clamp\)", k), find(r"const int cnt = min\(kB16", k)),
    "group loop": (find(r"const int cnt = min\(kB16", k), find(r"unsigned long long ev = 0, bl = 0;", k)),
    "epilogue": (find(r"unsigned long long ev = 0, bl = 0;", k), find(r"^template <int KIND, int ORDER, int MODE>", k)),
}
hdr = next(r for r in rows if r and r[0] == "Line No")
si, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
cur, agg = None, {}
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > ii and r[0] not in ("", "Line No", "Function Name") and r[2] == "-":
        ln = int(r[0])
        if cur == "blend.cu":
            reg = next((n for n, (a, b) in ranges.items() if a <= ln < b), "kernel body")
        elif cur.startswith("tile_sort"):
            reg = "sort"
        elif cur.startswith("sm_100_rt"):
            reg = "walk"  # the packed f32x2 builtins (__ffma2_rn ...) the walk is made of
        else:
            reg = "other:" + cur
        a = agg.setdefault(reg, [0, 0])
        a[0] += int(r[si] or 0)
        a[1] += int(r[ii] or 0)
ts = sum(a[0] for a in agg.values()) or 1
ti = sum(a[1] for a in agg.values()) or 1
print(f"total: {ti / 1e6:.1f}M warp instructions, {ts} stall samples")
for n, (s_, i_) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:34s} instr {i_ / 1e6:6.1f}M ({100 * i_ / ti:4.1f}%)  stalls {100 * s_ / ts:5.1f}%")
