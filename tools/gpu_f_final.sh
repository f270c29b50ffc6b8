# c2 / c4 bench lines (with cpu baseline and parity) and ncu captures after the a5 changes
O=gpurun_out/ff; mkdir -p $O; rm -f $O/*
for c in c2 c4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --graph > $O/bench_$c.log 2>&1; echo "bench_$c=$?" >> $O/status.txt; done
prof () {
  B="python bench.py --config $2 --steps 1 --warmup 3 --no-e2e --no-cpu"
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"$3" -s 1 -c 1 -o /tmp/prof_$1 $B > $O/ncu_$1.log 2>&1
  echo "ncu_$1=$?" >> $O/status.txt
  ncu -i /tmp/prof_$1.ncu-rep --page raw --csv > $O/prof_$1_raw.csv 2>/dev/null
  ncu -i /tmp/prof_$1.ncu-rep --page details --csv > $O/prof_$1_details.csv 2>/dev/null
  ncu -i /tmp/prof_$1.ncu-rep --page source --csv --print-source cuda,sass > $O/prof_$1_src.csv 2>/dev/null
  gzip -f $O/prof_$1_src.csv
}
prof c2 c2 "bm_boxf"
prof c4 c4 "bm_boxf"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/status.txt
