O=gpurun_out/hp2; mkdir -p $O; rm -f $O/*
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --graph > $O/bench_c3.log 2>&1; echo "bench_c3=$?" >> $O/status.txt
timeout 600 python bench.py --config c3 --metric ncc --steps 5 --warmup 3 --no-e2e > $O/bench_ncc_c3.log 2>&1; echo "ncc_c3=$?" >> $O/status.txt
timeout 600 python bench.py --config c3 --kernel boxf --steps 5 --warmup 3 --no-e2e --no-cpu > $O/bench_boxf_c3.log 2>&1; echo "boxf_c3=$?" >> $O/status.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > $O/pytest_gpu.log 2>&1; echo "pytest=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/status.txt
