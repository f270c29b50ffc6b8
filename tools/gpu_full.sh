mkdir -p gpurun_out
rm -f gpurun_out/full_status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> gpurun_out/full_status.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/full_status.txt
for c in c3 c2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_d_$c.log 2>&1; echo "bench_$c=$?" >> gpurun_out/full_status.txt; done
