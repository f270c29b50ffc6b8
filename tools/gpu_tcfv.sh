# tcf variants on c3 (bench) + phase counters + tcf tests with the default build. Outputs gpurun_out/tcfv/.
O=gpurun_out/tcfv; mkdir -p $O; rm -f $O/*
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_main.log 2>&1
for v in ${VARS:-nb s1 nbs1}; do
  SCBM_LIB=paper_2006_13714_b200/build/var_$v/libscbm.so timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_$v.log 2>&1
done
for v in ${PVARS:-tp tpnb}; do
SCBM_LIB=paper_2006_13714_b200/build/var_$v/libscbm.so timeout 300 python -c "
import torch, numpy as np
from paper_2006_13714_b200 import bm, synth
cfg = synth.config_by_name('c3')
x = torch.from_numpy(synth.make_input(cfg, 1)).cuda()
p = bm.Plan(cfg.H, cfg.W, cfg.C, cfg.b, cfg.s, cfg.Wn, cfg.K, cfg.dtype)
p.run(x); torch.cuda.synchronize()
" > $O/$v.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x -k "${PYK:-tcf or c3 or full}" > $O/pytest.log 2>&1; echo "pytest=$?" >> $O/status.txt
