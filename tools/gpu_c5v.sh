# c5 box-kernel variants: bench each (interleaved twice), box / temporal / packed tests on the sentinel build
O=gpurun_out/c5v; mkdir -p $O; rm -f $O/*
for r in 1 2; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > $O/bench_main_$r.log 2>&1
for v in ${VARS:-sent np3 np4 np7}; do
  SCBM_LIB=paper_2006_13714_b200/build/var_$v/libscbm.so timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > $O/bench_${v}_$r.log 2>&1
done
done
SCBM_LIB=paper_2006_13714_b200/build/var_sent/libscbm.so timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x -k "box or c5 or c1 or temporal or packed or stress or random" > $O/pytest_sent.log 2>&1; echo "pytest=$?" >> $O/status.txt
