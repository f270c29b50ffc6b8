# Round-2 first call: tcgen05 peaks, full-table parity tests, c5 bench with the parity field,
# ncu capture of the tensor-core matcher on c5.
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2006_13714_b200/csrc -o tools/tc_peaks tools/tc_peaks.cu
timeout 120 tools/tc_peaks > gpurun_out/tc_peaks.json 2> gpurun_out/tc_peaks.err; echo "tc_peaks=$?" > gpurun_out/status.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x -k "full" > gpurun_out/pytest_full.log 2>&1; echo "pytest_full=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c5.log 2>&1; echo "bench=$?" >> gpurun_out/status.txt
B="python bench.py --config c5 --kernel tc --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 300 $B > gpurun_out/plain_tc.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bm_tc" -s 2 -c 1 -o gpurun_out/prof_tc_c5 $B > gpurun_out/ncu_tc.log 2>&1; echo "ncu_tc=$?" >> gpurun_out/status.txt
