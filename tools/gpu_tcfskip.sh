cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tskip; rm -f gpurun_out/tskip/*
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/tskip/base.log 2>&1
for v in 1 2 4 6; do SCBM_LIB=paper_2006_13714_b200/build/var_tskip$v/libscbm.so timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/tskip/v$v.log 2>&1; done
