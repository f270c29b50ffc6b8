# tcf bound sweep: tcf / c3 tests, c3 bench, per-phase cycle counters. Outputs gpurun_out/bound/.
O=gpurun_out/bound; mkdir -p $O; rm -f $O/*
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_c3.log 2>&1; echo "bench=$?" >> $O/status.txt
SCBM_LIB=paper_2006_13714_b200/build/var_tprof/libscbm.so timeout 300 python -c "
import torch, numpy as np
from paper_2006_13714_b200 import bm, synth
cfg = synth.config_by_name('c3')
x = torch.from_numpy(synth.make_input(cfg, 1)).cuda()
p = bm.Plan(cfg.H, cfg.W, cfg.C, cfg.b, cfg.s, cfg.Wn, cfg.K, cfg.dtype)
p.run(x); torch.cuda.synchronize()
" > $O/tprof.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x -k "tcf or c3 or full" > $O/pytest.log 2>&1; echo "pytest=$?" >> $O/status.txt
