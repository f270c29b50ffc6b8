# After restricting the tile-height choice to 1-CTA/SM launches: the float lines and the boxf tests.
O=gpurun_out/r2h
mkdir -p $O; rm -f $O/*
for c in m1 v1 c4 c2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.log 2>&1; echo "bench_$c=$?" >> $O/status.txt; done
timeout 600 python bench.py --config c4 --metric ncc --steps 5 --warmup 3 --no-e2e > $O/bench_ncc_c4.log 2>&1; echo "ncc_c4=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/status.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 > $O/pytest_gpu.log 2>&1; echo "pytest=$?" >> $O/status.txt
