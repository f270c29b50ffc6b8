# Bench tuning variants of the library on one config:  VARS="m3 shfl" CONFIG=c5 bash tools/variants.sh
mkdir -p gpurun_out
B="python bench.py --config ${CONFIG:-c5} --steps 5 --warmup 3 --no-e2e --no-cpu"
timeout 300 $B > gpurun_out/var_default.log 2>&1
for v in $VARS; do
  SCBM_LIB=paper_2006_13714_b200/build/var_$v/libscbm.so timeout 300 $B > gpurun_out/var_$v.log 2>&1
  if [ -n "$VTEST" ]; then SCBM_LIB=paper_2006_13714_b200/build/var_$v/libscbm.so timeout 600 python -m pytest tests -m gpu -q -x -k "$VTEST" > gpurun_out/var_${v}_test.log 2>&1; fi
done
