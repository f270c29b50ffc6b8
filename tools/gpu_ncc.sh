mkdir -p gpurun_out
rm -f gpurun_out/ncc_status.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -k "ncc" > gpurun_out/pytest_ncc.log 2>&1; echo "ncc=$?" >> gpurun_out/ncc_status.txt
for c in c3 c4; do timeout 300 python bench.py --config $c --metric ncc --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ncc_$c.log 2>&1; echo "bench_$c=$?" >> gpurun_out/ncc_status.txt; done
