# ncu source-level capture of K3 at C3 (6M splats, 4K)
bash tools/ncu_kernel.sh k_duplicate_buckets r02_k3c3_src --workload c3 > /dev/null 2>&1
python tools/src_report.py gpurun_out/r02_k3c3_src_src.csv 25 > gpurun_out/r02_k3c3_lines.txt 2>&1
head -27 gpurun_out/r02_k3c3_lines.txt
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r02_k3c3_src_raw.csv'))); hdr=rows[0]; r=rows[2]
for w in ['gpu__time_duration.sum','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_sector_hit_rate.pct']:
    print(w, r[hdr.index(w)] if w in hdr else None)
st=[(h, float(r[i])) for i,h in enumerate(hdr) if h.startswith('smsp__average_warps_issue_stalled') and h.endswith('per_issue_active.ratio')]
st.sort(key=lambda x:-x[1]); print([ (h.split('stalled_')[1].split('_per')[0], round(v,2)) for h,v in st[:8]])
PY
