mkdir -p gpurun_out
rm -f gpurun_out/boxf_status.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -k "boxf or c2 or c3_c4 or f32 or nlm or ncc" > gpurun_out/pytest_boxf.log 2>&1; echo "pytest=$?" >> gpurun_out/boxf_status.txt
for c in c2 c3 c4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_boxf_$c.log 2>&1; echo "bench_$c=$?" >> gpurun_out/boxf_status.txt; done
for c in c3 c4; do timeout 300 python bench.py --config $c --metric ncc --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ncc_$c.log 2>&1; echo "ncc_$c=$?" >> gpurun_out/boxf_status.txt; done
