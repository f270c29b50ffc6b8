cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sift; rm -f gpurun_out/sift/*
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tcf or tc_f32 or c3_c4_full" > gpurun_out/sift/pytest.log 2>&1; echo "pytest=$?" >> gpurun_out/sift/status
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/sift/new.log 2>&1
SCBM_LIB=paper_2006_13714_b200/build/var_a5old/libscbm.so timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/sift/old.log 2>&1
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/sift/new2.log 2>&1
