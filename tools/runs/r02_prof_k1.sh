# ncu source-level captures of K1 (fused preprocess), K3 and K2 at C2 poly1
bash tools/ncu_kernel.sh k_preprocess r02_k1_src > /dev/null 2>&1
python tools/src_report.py gpurun_out/r02_k1_src_src.csv 60 > gpurun_out/r02_k1_lines.txt 2>&1
bash tools/ncu_kernel.sh k_duplicate_buckets r02_k3_src > /dev/null 2>&1
python tools/src_report.py gpurun_out/r02_k3_src_src.csv 30 > gpurun_out/r02_k3_lines.txt 2>&1
bash tools/ncu_kernel.sh k_tile_scan r02_k2_src > /dev/null 2>&1
python tools/src_report.py gpurun_out/r02_k2_src_src.csv 20 > gpurun_out/r02_k2_lines.txt 2>&1
head -64 gpurun_out/r02_k1_lines.txt; head -32 gpurun_out/r02_k3_lines.txt; head -22 gpurun_out/r02_k2_lines.txt
