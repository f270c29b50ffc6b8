# ncu full capture of the box-sum matcher (and the norm kernel) on c5, after a plain run exits 0.
mkdir -p gpurun_out
B="python bench.py --config ${CONFIG:-c5} --kernel ${KERNEL:-box} --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 300 $B > gpurun_out/plain_box.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-bm_box|norm_direct}" -s 2 -c 2 -o gpurun_out/prof_box $B > gpurun_out/ncu_box.log 2>&1
echo "rc=$?" > gpurun_out/prof_status.txt
