"""Run one float box-kernel case (for compute-sanitizer):  python tools/boxf_case.py s b H W Wn K"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2006_13714_b200 import synth  # noqa: E402
from paper_2006_13714_b200.bm import SC_KERNEL_BOXF, Plan  # noqa: E402

s, b, H, W, Wn, K = map(int, sys.argv[1:7])
rng = np.random.Generator(np.random.PCG64(1))
x = synth.random_image(rng, 2, 1, H, W, "f32")
p = Plan(H, W, 1, b, s, Wn, K, "f32")
p.set_kernel(SC_KERNEL_BOXF)
idx, dist = p.run(torch.from_numpy(x).cuda())
torch.cuda.synchronize()
print("ok", idx.shape)
