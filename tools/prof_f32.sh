# f32 configs: bench lines + ncu full capture of the default matcher on c3 and c4.
mkdir -p gpurun_out
for c in c2 c3 c4; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$c.log 2>&1; done
for c in ${PCONF:-c3 c4}; do
  B="python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bm_" -s 1 -c 1 -o gpurun_out/prof_$c $B > gpurun_out/ncu_$c.log 2>&1
done
