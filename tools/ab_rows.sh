set -x
mkdir -p gpurun_out/ab
for cfg in c4 c2 v1 m1; do
  for R in 8 auto; do
    if [ $R = auto ]; then unset SC_BM_BOXF_ROWS; else export SC_BM_BOXF_ROWS=$R; fi
    timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/ab/${cfg}_$R.jsonl 2> gpurun_out/ab/${cfg}_$R.err
  done
done
for R in 8 auto; do
  if [ $R = auto ]; then unset SC_BM_BOXF_ROWS; else export SC_BM_BOXF_ROWS=$R; fi
  timeout 300 python bench.py --config c4 --metric ncc --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/ab/ncc_c4_$R.jsonl 2> gpurun_out/ab/ncc_c4_$R.err
done
unset SC_BM_BOXF_ROWS
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "boxf or c2_full or c3_c4_full or ncc or bm3d" > gpurun_out/ab/pytest.log 2>&1
echo pytest exit $?
