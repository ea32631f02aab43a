# ncu source-level capture of the C2 blend (poly1) + region summary, and a full capture of K1/K3
bash tools/ncu_kernel.sh blend16 r02_blend_src > /dev/null 2>&1
python tools/src_regions.py gpurun_out/r02_blend_src_src.csv > gpurun_out/r02_blend_regions.txt 2>&1
python tools/src_report.py gpurun_out/r02_blend_src_src.csv 50 >> gpurun_out/r02_blend_regions.txt 2>&1
cat gpurun_out/r02_blend_regions.txt | head -70
