mkdir -p gpurun_out
for c in ${CONFIGS:-c2 c3}; do
B="python bench.py --config $c --kernel tcf --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 300 $B > gpurun_out/plain_tcf_$c.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bm_tcf" -s 2 -c 1 -o gpurun_out/prof_tcf_$c $B > gpurun_out/ncu_tcf_$c.log 2>&1
echo "$c=$?" >> gpurun_out/prof_tcf_status.txt
done
