# FFMA2 float box kernel: peaks, float tests, c2/c4 bench with and without FFMA2. Outputs gpurun_out/f2/.
O=gpurun_out/f2; mkdir -p $O; rm -f $O/*
tools/peaks > $O/peaks.json 2>&1
for c in c2 c4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_$c.log 2>&1
  SCBM_LIB=paper_2006_13714_b200/build/var_f2off/libscbm.so timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_${c}_off.log 2>&1
done
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x -k "boxf or c2 or c4 or float or f32" > $O/pytest.log 2>&1; echo "pytest=$?" >> $O/status.txt
