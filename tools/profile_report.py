"""Writes the round's profile summary (markdown) from the ncu outputs that
tools/collect_profiles.sh brings back:

  python tools/profile_report.py ROUND gpurun_out/prof_launches_c2.csv \
      gpurun_out/prof_launches_c2_exp.csv --raw gpurun_out/prof_full_c2_raw.csv > profiles/rNN_summary.md

Launch lists are ncu `gpu__time_duration.sum --clock-control none` passes
(cold caches, serialised launches): the per-kernel SHARE of a frame is the
comparable quantity, not the absolute time. The raw page gives per-kernel DRAM
traffic (the roofline `traffic` field) and instruction counts."""
import argparse
import csv
import re


def frame_launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    frames, cur = [], []
    for r in rows[hi + 1:]:
        name = re.sub(r"\(.*", "", r[ki].replace("(anonymous namespace)::", "").replace("unnamed>::", ""))
        if ("k_preprocess" in name or "k_geometry" in name) and cur:
            frames.append(cur)
            cur = []
        cur.append((name, float(r[vi].replace(",", "")) / 1000.0))
    frames.append(cur)
    return frames[-1]


def raw_metrics(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    want = {
        "gpu__time_duration.sum": "time",
        "dram__bytes_read.sum": "dram_rd",
        "dram__bytes_write.sum": "dram_wr",
        "smsp__inst_executed.sum": "inst",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy",
        "sm__inst_executed.avg.per_cycle_active": "ipc",
        "launch__registers_per_thread": "regs",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu",
    }
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
    out = []
    for r in rows[2:]:
        d = {"name": re.sub(r"\(.*", "", r[hdr.index("Kernel Name")].replace("(anonymous namespace)::", "").replace("unnamed>::", ""))}
        for k, short in want.items():
            if k in hdr:
                i = hdr.index(k)
                v = float(r[i].replace(",", ""))
                d[short] = v * scale.get(units[i], 1.0)
        out.append(d)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("round")
    ap.add_argument("launch_lists", nargs="+")
    ap.add_argument("--raw")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    print(f"# Profile summary, round {a.round}\n")
    if a.note:
        print(a.note + "\n")
    for p in a.launch_lists:
        f = frame_launches(p)
        tot = sum(v for _, v in f)
        agg = {}
        for n, v in f:
            agg[n] = agg.get(n, 0.0) + v
        print(f"## Launch list `{p.split('/')[-1]}` (last frame, ncu cold/serialised)\n")
        print("| kernel | µs | share |\n|---|---:|---:|")
        for n, v in sorted(agg.items(), key=lambda x: -x[1]):
            print(f"| `{n}` | {v:.1f} | {100 * v / tot:.1f}% |")
        print(f"| **total ({len(f)} launches)** | {tot:.1f} | |\n")
    if a.raw:
        print(f"## `ncu --set full` per-kernel metrics (`{a.raw.split('/')[-1]}`)\n")
        print("| kernel | µs | DRAM read MB | DRAM write MB | DRAM GB/s | warp instr (M) | regs | occupancy % |")
        print("|---|---:|---:|---:|---:|---:|---:|---:|")
        for d in raw_metrics(a.raw):
            t = d.get("time", 0.0)
            mb = d.get("dram_rd", 0.0) + d.get("dram_wr", 0.0)
            print(f"| `{d['name']}` | {t:.1f} | {d.get('dram_rd', 0):.1f} | {d.get('dram_wr', 0):.1f} | "
                  f"{mb / t * 1e3 if t else 0:.0f} | {d.get('inst', 0) / 1e6:.1f} | "
                  f"{d.get('regs', 0):.0f} | {d.get('occupancy', 0):.1f} |")
        print()
        print("Pipe utilisation (% of peak, active cycles) — the north star's FP32-FMA evidence for the blend:\n")
        print("| kernel | issue slots | FMA pipe (FFMA/FFMA2/FMUL) | ALU | FP64 | XU (MUFU, conversions) | LSU |")
        print("|---|---:|---:|---:|---:|---:|---:|")
        for d in raw_metrics(a.raw):
            print(f"| `{d['name']}` | {d.get('issue', 0):.1f} | {d.get('fma', 0):.1f} | {d.get('alu', 0):.1f} | "
                  f"{d.get('fp64', 0):.1f} | {d.get('xu', 0):.1f} | {d.get('lsu', 0):.1f} |")
        print()


if __name__ == "__main__":
    main()
