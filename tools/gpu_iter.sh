# One iteration: selected GPU tests, c5 bench of the given kernels, ncu capture of the box kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "${PYTEST_K:-box or r32 or c5 or c1 or lanes}" > gpurun_out/pytest_quick.log 2>&1; echo "pytest=$?" > gpurun_out/quick_status.txt
for k in ${KERNELS:-box}; do
  timeout 300 python bench.py --config ${CONFIG:-c5} --kernel $k --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_q_$k.log 2>&1; echo "bench_$k=$?" >> gpurun_out/quick_status.txt
done
if [ -n "$PROF" ]; then
  B="python bench.py --config ${CONFIG:-c5} --kernel box --steps 1 --warmup 3 --no-e2e --no-cpu"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bm_box" -s 2 -c 1 -o gpurun_out/prof_box $B > gpurun_out/ncu_box.log 2>&1
  echo "prof=$?" >> gpurun_out/quick_status.txt
fi
