mkdir -p gpurun_out
rm -f gpurun_out/c5_status.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "${PYTEST_K:-box or c5 or temporal}" > gpurun_out/pytest_c5.log 2>&1; echo "pytest=$?" >> gpurun_out/c5_status.txt
for i in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c5_$i.log 2>&1; echo "bench_$i=$?" >> gpurun_out/c5_status.txt; done
