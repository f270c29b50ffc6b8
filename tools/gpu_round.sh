# Full round evidence: smoke, all GPU tests, deliverables (bench/reference/torchrun/launches/ncu of the
# c5 matcher) and per-config bench lines + ncu captures of the f32 matchers.
mkdir -p gpurun_out
bash tools/gpu_all.sh
for c in c1 c2 c3 c4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --graph > gpurun_out/bench_$c.log 2>&1; echo "bench_$c=$?" >> gpurun_out/status.txt; done
CONFIGS="c2 c3 c4" bash tools/prof_cfg.sh
