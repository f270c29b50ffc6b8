mkdir -p gpurun_out
rm -f gpurun_out/tcf_status.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -k "tcf" > gpurun_out/pytest_tcf.log 2>&1; echo "tcf=$?" >> gpurun_out/tcf_status.txt
for c in c2 c3; do timeout 300 python bench.py --config $c --kernel tcf --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_tcf_$c.log 2>&1; echo "bench_$c=$?" >> gpurun_out/tcf_status.txt; done
