O=gpurun_out/hp; mkdir -p $O; rm -f $O/*
for r in 1 2; do
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_main_$r.log 2>&1
for v in hpw old4; do
SCBM_LIB=paper_2006_13714_b200/build/var_$v/libscbm.so timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_${v}_$r.log 2>&1
done; done
timeout 600 python bench.py --config c3 --kernel boxf --steps 5 --warmup 3 --no-e2e --no-cpu > $O/bench_boxf_c3.log 2>&1; echo "boxf_c3=$?" >> $O/status.txt
timeout 600 python bench.py --config c3 --metric ncc --steps 5 --warmup 3 --no-e2e --no-cpu > $O/bench_ncc_c3.log 2>&1; echo "ncc_c3=$?" >> $O/status.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x -k "boxf or c3 or ncc or tcf or full or fixup" > $O/pytest.log 2>&1; echo "pytest=$?" >> $O/status.txt
