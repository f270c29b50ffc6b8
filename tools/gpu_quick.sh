# Quick GPU iteration: selected GPU tests (PYTEST_K) + c5 bench lines for the given kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "${PYTEST_K:-box or r32 or c5 or c1 or lanes}" > gpurun_out/pytest_quick.log 2>&1; echo "pytest=$?" > gpurun_out/quick_status.txt
for k in ${KERNELS:-box}; do
  timeout 300 python bench.py --config ${CONFIG:-c5} --kernel $k --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_q_$k.log 2>&1; echo "bench_$k=$?" >> gpurun_out/quick_status.txt
done
