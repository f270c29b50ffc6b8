# Evidence for the float box kernel's tile-height choice (boxf_rows): smoke, the whole GPU suite,
# the default c5 line, c4 / m1 / NCC c4 lines, an ncu --set full capture of the c4 matcher.
O=gpurun_out/r2g
mkdir -p $O; rm -f $O/*
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/status.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 > $O/pytest_gpu.log 2>&1; echo "pytest=$?" >> $O/status.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c5.log 2>&1; echo "bench_c5=$?" >> $O/status.txt
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --graph > $O/bench_c4.log 2>&1; echo "bench_c4=$?" >> $O/status.txt
timeout 600 python bench.py --config m1 --steps 10 --warmup 3 > $O/bench_m1.log 2>&1; echo "bench_m1=$?" >> $O/status.txt
timeout 600 python bench.py --config c4 --metric ncc --steps 5 --warmup 3 --no-e2e > $O/bench_ncc_c4.log 2>&1; echo "ncc_c4=$?" >> $O/status.txt
B="python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"bm_boxf" -s 1 -c 1 -o /tmp/prof_c4 $B > $O/ncu_c4.log 2>&1
echo "ncu_c4=$?" >> $O/status.txt
ncu -i /tmp/prof_c4.ncu-rep --page raw --csv > $O/prof_c4_raw.csv 2>/dev/null
ncu -i /tmp/prof_c4.ncu-rep --page details --csv > $O/prof_c4_details.csv 2>/dev/null
ncu -i /tmp/prof_c4.ncu-rep --page source --csv --print-source cuda,sass > $O/prof_c4_src.csv 2>/dev/null
gzip -f $O/prof_c4_src.csv
