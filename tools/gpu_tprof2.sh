O=gpurun_out/tprof2; mkdir -p $O; rm -f $O/*
for v in tprof tprof0; do
SCBM_LIB=paper_2006_13714_b200/build/var_$v/libscbm.so timeout 300 python -c "
import torch, numpy as np
from paper_2006_13714_b200 import bm, synth
cfg = synth.config_by_name('c3')
x = torch.from_numpy(synth.make_input(cfg, 1)).cuda()
p = bm.Plan(cfg.H, cfg.W, cfg.C, cfg.b, cfg.s, cfg.Wn, cfg.K, cfg.dtype)
p.run(x); torch.cuda.synchronize()
" > $O/$v.log 2>&1
done
