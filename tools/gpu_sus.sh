O=gpurun_out/sus; mkdir -p $O; rm -f $O/*
for r in 1 2; do
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_main_$r.log 2>&1
SCBM_LIB=paper_2006_13714_b200/build/var_nosus/libscbm.so timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_nosus_$r.log 2>&1
done
timeout 300 python bench.py --config c2 --kernel tcf --steps 10 --warmup 3 --no-e2e --no-cpu > $O/bench_tcf_c2.log 2>&1
timeout 300 python bench.py --kernel tc --steps 2 --warmup 3 --no-e2e --no-cpu > $O/bench_tc_c5.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x -k "tcf or c3 or tc_" > $O/pytest.log 2>&1; echo "pytest=$?" >> $O/status.txt
