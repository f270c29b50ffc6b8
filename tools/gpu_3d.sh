mkdir -p gpurun_out
rm -f gpurun_out/s3d_status.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -k "bm3d" > gpurun_out/pytest_3d.log 2>&1; echo "pytest=$?" >> gpurun_out/s3d_status.txt
for c in v1 m1; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.log 2>&1; echo "bench_$c=$?" >> gpurun_out/s3d_status.txt; done
