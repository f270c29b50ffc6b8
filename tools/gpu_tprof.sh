cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tprof; rm -f gpurun_out/tprof/*
SCBM_LIB=paper_2006_13714_b200/build/var_tprof/libscbm.so timeout 300 python -c "
import torch, numpy as np
from paper_2006_13714_b200 import bm, synth
cfg = synth.config_by_name('c3')
x = torch.from_numpy(synth.make_input(cfg, 1)).cuda()
p = bm.Plan(cfg.H, cfg.W, cfg.C, cfg.b, cfg.s, cfg.Wn, cfg.K, cfg.dtype)
print('kernel', p.info()['kernel'])
p.run(x); torch.cuda.synchronize()
" > gpurun_out/tprof/out.log 2>&1
