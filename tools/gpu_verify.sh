# final-build verification: smoke, the whole GPU suite, the default bench line and c3
O=gpurun_out/verify; mkdir -p $O; rm -f $O/*
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/status.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > $O/pytest_gpu.log 2>&1; echo "pytest=$?" >> $O/status.txt
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "bench=$?" >> $O/status.txt
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 > $O/bench_c3.log 2>&1; echo "bench_c3=$?" >> $O/status.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.log 2>&1; echo "ref=$?" >> $O/status.txt
