# Current-state check: smoke, the GPU suite, bench lines c5/c2/c3/c4. Outputs under gpurun_out/st/.
O=gpurun_out/st
mkdir -p $O; rm -f $O/*
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/status.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > $O/pytest_gpu.log 2>&1; echo "pytest=$?" >> $O/status.txt
for c in c5 c2 c3 c4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu > $O/bench_$c.log 2>&1; echo "bench_$c=$?" >> $O/status.txt; done
