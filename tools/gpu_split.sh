O=gpurun_out/split; mkdir -p $O; rm -f $O/*
for c in c4 c2; do
timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_$c.log 2>&1
SCBM_LIB=paper_2006_13714_b200/build/var_nosplit/libscbm.so timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_${c}_nosplit.log 2>&1
done
timeout 300 python bench.py --config c4 --metric ncc --steps 5 --warmup 3 --no-e2e --no-cpu > $O/bench_ncc_c4.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x -k "boxf or c4 or c2 or full or float or ncc" > $O/pytest.log 2>&1; echo "pytest=$?" >> $O/status.txt
