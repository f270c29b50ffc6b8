# round deliverables: bench (default), reference arm, torchrun N=1, ncu launch list + full capture
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.log 2>&1; echo "bench=$?" > gpurun_out/deliv_status.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo "ref=$?" >> gpurun_out/deliv_status.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu --gather > gpurun_out/bench_torchrun1.log 2>&1; echo "torchrun=$?" >> gpurun_out/deliv_status.txt
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 300 $B > gpurun_out/plain_launch.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "launches=$?" >> gpurun_out/deliv_status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bm_box" -s 2 -c 1 -o gpurun_out/prof_default $B > gpurun_out/ncu_full.log 2>&1; echo "ncufull=$?" >> gpurun_out/deliv_status.txt
