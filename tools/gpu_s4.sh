O=gpurun_out/tcfv; mkdir -p $O; rm -f $O/*
for r in 1 2; do
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_main_$r.log 2>&1
SCBM_LIB=paper_2006_13714_b200/build/var_s4/libscbm.so timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_s4_$r.log 2>&1
done
for v in tp s4p; do
SCBM_LIB=paper_2006_13714_b200/build/var_$v/libscbm.so timeout 300 python -c "
import torch, numpy as np
from paper_2006_13714_b200 import bm, synth
cfg = synth.config_by_name('c3')
x = torch.from_numpy(synth.make_input(cfg, 1)).cuda()
p = bm.Plan(cfg.H, cfg.W, cfg.C, cfg.b, cfg.s, cfg.Wn, cfg.K, cfg.dtype)
p.run(x); torch.cuda.synchronize()
" > $O/$v.log 2>&1
done
SCBM_LIB=paper_2006_13714_b200/build/var_s4/libscbm.so timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x -k "tcf or c3 or full" > $O/pytest_s4.log 2>&1; echo "pytest=$?" >> $O/status.txt
