O=gpurun_out/fill; mkdir -p $O; rm -f $O/*
for r in 1 2; do
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_main_$r.log 2>&1
SCBM_LIB=paper_2006_13714_b200/build/var_nofill/libscbm.so timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_nofill_$r.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x -k "tcf or c3 or full" > $O/pytest.log 2>&1; echo "pytest=$?" >> $O/status.txt
