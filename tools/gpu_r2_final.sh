# Round-2 final evidence: smoke, the whole GPU suite, bench lines (every config, NCC, 3D, next rows,
# tensor-core matchers, reference arm, torchrun N=1 with the gathers), the c5 launch list and ncu
# captures (CSV exports) of the c5 box kernel and the c2/c3/c4 float matchers. Outputs gpurun_out/r2f/.
O=gpurun_out/r2f
mkdir -p $O; rm -f $O/*
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/status.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > $O/pytest_gpu.log 2>&1; echo "pytest=$?" >> $O/status.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c5.log 2>&1; echo "bench_c5=$?" >> $O/status.txt
for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --graph > $O/bench_$c.log 2>&1; echo "bench_$c=$?" >> $O/status.txt; done
timeout 600 python bench.py --config c2 --kernel tcf --steps 5 --warmup 3 --no-e2e --no-cpu > $O/bench_tcf_c2.log 2>&1; echo "tcf_c2=$?" >> $O/status.txt
timeout 600 python bench.py --config c3 --kernel boxf --steps 5 --warmup 3 --no-e2e --no-cpu > $O/bench_boxf_c3.log 2>&1; echo "boxf_c3=$?" >> $O/status.txt
timeout 600 python bench.py --kernel tc --steps 2 --warmup 3 --no-e2e --no-cpu > $O/bench_tc_c5.log 2>&1; echo "tc_c5=$?" >> $O/status.txt
for c in c5 c2 c3 c4; do timeout 600 python bench.py --config $c --metric ncc --steps 5 --warmup 3 --no-e2e > $O/bench_ncc_$c.log 2>&1; echo "ncc_$c=$?" >> $O/status.txt; done
for c in v1 m1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.log 2>&1; echo "bench_$c=$?" >> $O/status.txt; done
timeout 600 python bench.py --temporal 1 --steps 5 --warmup 3 --no-cpu > $O/bench_temporal_c5.log 2>&1; echo "temporal=$?" >> $O/status.txt
for op in group nlm nlm_avg; do timeout 600 python bench.py --config c2 --op $op --steps 5 --warmup 3 > $O/bench_${op}_c2.log 2>&1; echo "${op}=$?" >> $O/status.txt; done
timeout 600 python bench.py --op group --steps 5 --warmup 3 > $O/bench_group_c5.log 2>&1; echo "group_c5=$?" >> $O/status.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.log 2>&1; echo "ref=$?" >> $O/status.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu --gather > $O/bench_torchrun1.log 2>&1; echo "torchrun=$?" >> $O/status.txt
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 300 $B > $O/plain_launch.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv $B > $O/ncu_launch.log 2>&1; echo "launches=$?" >> $O/status.txt
# ncu --set full captures, CSV exports only (gpurun_out <= 64 MiB)
prof () {  # name config kernel-regex extra
  B="python bench.py --config $2 --steps 1 --warmup 3 --no-e2e --no-cpu $4"
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"$3" -s 1 -c 1 -o /tmp/prof_$1 $B > $O/ncu_$1.log 2>&1
  echo "ncu_$1=$?" >> $O/status.txt
  ncu -i /tmp/prof_$1.ncu-rep --page raw --csv > $O/prof_$1_raw.csv 2>/dev/null
  ncu -i /tmp/prof_$1.ncu-rep --page details --csv > $O/prof_$1_details.csv 2>/dev/null
  ncu -i /tmp/prof_$1.ncu-rep --page source --csv --print-source cuda,sass > $O/prof_$1_src.csv 2>/dev/null
  gzip -f $O/prof_$1_src.csv
}
prof c5 c5 "bm_box_kernel" ""
prof c2 c2 "bm_boxf" ""
prof c3 c3 "bm_tcf" ""
prof c4 c4 "bm_boxf" ""
