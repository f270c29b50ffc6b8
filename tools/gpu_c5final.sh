# c5 evidence after the sentinel rounds: bench (default line), gather paths at N = 1, launch list, ncu capture
O=gpurun_out/c5g; mkdir -p $O; rm -f $O/*
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/status.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c5.log 2>&1; echo "bench_c5=$?" >> $O/status.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --gather > $O/bench_gather1.log 2>&1; echo "gather1=$?" >> $O/status.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu --gather > $O/bench_torchrun1.log 2>&1; echo "torchrun=$?" >> $O/status.txt
timeout 600 python bench.py --temporal 1 --steps 5 --warmup 3 --no-cpu > $O/bench_temporal_c5.log 2>&1; echo "temporal=$?" >> $O/status.txt
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv $B > $O/ncu_launch.log 2>&1; echo "launches=$?" >> $O/status.txt
B="python bench.py --config c5 --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"bm_box_kernel" -s 1 -c 1 -o /tmp/prof_c5 $B > $O/ncu_c5.log 2>&1; echo "ncu_c5=$?" >> $O/status.txt
ncu -i /tmp/prof_c5.ncu-rep --page raw --csv > $O/prof_c5_raw.csv 2>/dev/null
ncu -i /tmp/prof_c5.ncu-rep --page details --csv > $O/prof_c5_details.csv 2>/dev/null
ncu -i /tmp/prof_c5.ncu-rep --page source --csv --print-source cuda,sass > $O/prof_c5_src.csv 2>/dev/null
gzip -f $O/prof_c5_src.csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x -k "box or c5 or c1 or temporal or packed or peer or ncc" > $O/pytest.log 2>&1; echo "pytest=$?" >> $O/status.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > $O/pytest_gpu_all.log 2>&1; echo "pytest_all=$?" >> $O/status.txt
