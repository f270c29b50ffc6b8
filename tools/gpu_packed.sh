set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pk
timeout 600 python -m pytest tests/test_packed.py -q -m gpu -x > gpurun_out/pk/pytest.log 2>&1; echo "pytest=$?" >> gpurun_out/pk/status
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/pk/bench_c5.log 2>&1; echo "bench=$?" >> gpurun_out/pk/status
