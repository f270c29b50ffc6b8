# bench every config with each CUDA-core kernel (no e2e / cpu legs)
mkdir -p gpurun_out
for k in ${KERNELS:-box simt warp}; do for c in ${CONFIGS:-c5 c1 c2 c3 c4}; do
  timeout 600 python bench.py --config $c --kernel $k --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_${k}_$c.log 2>&1
done; done
