# ncu full capture of the default matcher for CONFIG (after a plain run exits 0)
mkdir -p gpurun_out
for c in ${CONFIGS:-c3}; do
  B="python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu"
  timeout 300 $B > gpurun_out/plain_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bm_" -s 1 -c 1 -o gpurun_out/prof_$c $B > gpurun_out/ncu_$c.log 2>&1
done
