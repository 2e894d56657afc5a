import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_1811_00901_b200 import spin
from synth import clouds
for seed in (91, 2):
    P, Nn = clouds.bumpy_sphere(100000, seed)
    cen = torch.arange(100000, dtype=torch.int32, device='cuda')
    eng = spin.SpinEngine(torch.from_numpy(P).cuda(), torch.from_numpy(Nn).cuda())
    print('seed', seed, 'absmax', float(np.linalg.norm(P, axis=1).max()))
    for mode in ('nearest',):
      for W,b,c in ((32,0.01,0.0),(16,0.02,0.5),(16,0.02,0.0),(16,0.02,-np.inf),(8,0.05,-np.inf)):
        _, st = eng.generate(cen, W, b, c, mode=mode, schedule='SS', stats=True)
        print(mode, W, b, c, 'G', st['G'], 'ms %.3f' % st['elapsed_ms'], 'dense', st['tiles_dense'], st['dense_rows'], 'cand', st['pairs_candidate'], 'suphot', st['tiles_support_hot'], 'mma', st['filter_mma'], flush=True)
    eng.close()
