import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2006_13714_b200 import synth
from paper_2006_13714_b200.bm import Plan3D
for (P, d, H, W, b, s, sz, Wn, c, K) in [(3, 2, 50, 49, 8, 2, 2, 1, 1, 4), (4, 2, 19, 63, 8, 2, 1, 5, 1, 8), (5, 1, 44, 76, 7, 1, 1, 12, 4, 9), (3,1,41,53,7,1,1,15,1,16)]:
    rng = np.random.Generator(np.random.PCG64(1))
    vol = synth.random_image(rng, 1, P, H, W, "f32")[0]
    p = Plan3D(H, W, d, b, s, Wn, sz, c, K)
    gi, gd = p.run(torch.from_numpy(vol).cuda()); torch.cuda.synchronize()
    gi, gd = gi.cpu().numpy(), gd.cpu().numpy()
    oi, od = oracle.bm3d(vol, d, b, s, sz, Wn, c, K)
    bad = np.argwhere((gi != oi) | (np.abs(gd - od) > 1e-5 * np.maximum(od, 1e-9)))
    print((P, d, H, W, b, s, sz, Wn, c, K), 'bad', len(bad), 'of', gi.size, 'fix', p.debug_fix_count())
    for t in bad[:4]:
        z, r, k = t
        print('  z', z, 'ref', r, 'k', k, 'gpu', gi[z, r, :6], gd[z, r, :6], 'oracle', oi[z, r, :6], od[z, r, :6])
