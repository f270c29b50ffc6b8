# GPU round-trip: peaks, smoke, GPU parity tests, per-config bench lines.
mkdir -p gpurun_out
./tools/peaks > gpurun_out/peaks.json 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" > gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
for c in ${CONFIGS:-c5 c1 c2 c3 c4}; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$c.log 2>&1; echo "bench_$c=$?" >> gpurun_out/status.txt; done
