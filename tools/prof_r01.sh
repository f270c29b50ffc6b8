mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
for c in c1 c2 c3 c4; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$c.log 2>&1; done
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bm_simt -s 2 -c 1 -o gpurun_out/prof_c5 $B > gpurun_out/ncu_full.log 2>&1
timeout 300 python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bm_simt -s 3 -c 1 -o gpurun_out/prof_c3 python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full_c3.log 2>&1
echo done
