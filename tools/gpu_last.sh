# final build: smoke, whole GPU suite, c3 / c5 bench lines, ncu captures of the c5 box kernel and the c3 matcher
O=gpurun_out/last; mkdir -p $O; rm -f $O/*
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/status.txt
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --graph > $O/bench_c3.log 2>&1; echo "bench_c3=$?" >> $O/status.txt
timeout 600 python bench.py --config c3 --metric ncc --steps 5 --warmup 3 --no-e2e > $O/bench_ncc_c3.log 2>&1; echo "ncc_c3=$?" >> $O/status.txt
prof () {  # name config kernel-regex
  B="python bench.py --config $2 --steps 1 --warmup 3 --no-e2e --no-cpu"
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"$3" -s 1 -c 1 -o /tmp/prof_$1 $B > $O/ncu_$1.log 2>&1
  echo "ncu_$1=$?" >> $O/status.txt
  ncu -i /tmp/prof_$1.ncu-rep --page raw --csv > $O/prof_$1_raw.csv 2>/dev/null
  ncu -i /tmp/prof_$1.ncu-rep --page details --csv > $O/prof_$1_details.csv 2>/dev/null
  ncu -i /tmp/prof_$1.ncu-rep --page source --csv --print-source cuda,sass > $O/prof_$1_src.csv 2>/dev/null
  gzip -f $O/prof_$1_src.csv
}
prof c5 c5 "bm_box_kernel"
prof c3 c3 "bm_tcf"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > $O/pytest_gpu.log 2>&1; echo "pytest=$?" >> $O/status.txt
