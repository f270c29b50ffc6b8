mkdir -p gpurun_out
B="python bench.py --config ${CONFIG:-c5} --kernel tc --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 300 $B > gpurun_out/plain_tc.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bm_tc -s 1 -c 1 -o gpurun_out/prof_tc $B > gpurun_out/ncu_tc.log 2>&1
