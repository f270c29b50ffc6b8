mkdir -p gpurun_out
for d in 0 1 2 3; do SCBM_TC_DEBUG=$d timeout 300 python bench.py --config c5 --kernel tc --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_tc_dbg$d.log 2>&1; done
