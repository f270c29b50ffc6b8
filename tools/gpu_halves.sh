O=gpurun_out/halves; mkdir -p $O; rm -f $O/*
for r in 1 2; do
for c in c4 c2; do
timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_${c}_main_$r.log 2>&1
SCBM_LIB=paper_2006_13714_b200/build/var_nohalves/libscbm.so timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_${c}_nohalves_$r.log 2>&1
done; done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x -k "boxf or c2 or c4 or full or float or f32 or random" > $O/pytest.log 2>&1; echo "pytest=$?" >> $O/status.txt
