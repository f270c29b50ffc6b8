mkdir -p gpurun_out
rm -f gpurun_out/cmp_status.txt
timeout 300 python bench.py --config c3 --kernel boxf --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/cmp_c3_boxf.log 2>&1; echo "c3boxf=$?" >> gpurun_out/cmp_status.txt
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/cmp_c3_tcf.log 2>&1; echo "c3tcf=$?" >> gpurun_out/cmp_status.txt
timeout 300 python bench.py --config c2 --kernel tcf --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/cmp_c2_tcf.log 2>&1; echo "c2tcf=$?" >> gpurun_out/cmp_status.txt
