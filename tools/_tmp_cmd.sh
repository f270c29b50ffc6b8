timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "ncc or NCC or fixup" 2>&1 | tail -5
for c in c5 c2; do
  echo -n "$c "; timeout 300 python bench.py --config $c --metric ncc --steps 5 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | tee gpurun_out/bench_ncc_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])"
done
