set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tcf
rm -f gpurun_out/tcf/*
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tcf or tc_f32 or c3_c4_full" > gpurun_out/tcf/pytest.log 2>&1; echo "pytest=$?" >> gpurun_out/tcf/status
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e > gpurun_out/tcf/bench_c3.log 2>&1; echo "c3=$?" >> gpurun_out/tcf/status
timeout 600 python bench.py --config c2 --kernel tcf --steps 10 --warmup 3 --no-e2e > gpurun_out/tcf/bench_tcf_c2.log 2>&1; echo "c2=$?" >> gpurun_out/tcf/status
