mkdir -p gpurun_out
rm -f gpurun_out/f_status.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x -k "boxf or c2 or c3_c4 or bm3d" > gpurun_out/pytest_f.log 2>&1; echo "pytest=$?" >> gpurun_out/f_status.txt
for c in c2 c3 c4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_f_$c.log 2>&1; echo "bench_$c=$?" >> gpurun_out/f_status.txt; done
