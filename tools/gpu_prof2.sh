# source-level ncu captures: float box kernel (c2, c4), c5 box kernel; CSV exports only
CONFIGS="c2 c4" bash tools/prof_f.sh
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 300 $B > gpurun_out/plain_c5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bm_box_kernel" -s 1 -c 1 -o /tmp/prof_c5 $B > gpurun_out/ncu_c5.log 2>&1
echo "c5=$?" >> gpurun_out/prof_f_status.txt
ncu -i /tmp/prof_c5.ncu-rep --page raw --csv > gpurun_out/prof_c5_raw.csv 2>/dev/null
ncu -i /tmp/prof_c5.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_c5_src.csv 2>/dev/null
gzip -f gpurun_out/prof_c5_src.csv
