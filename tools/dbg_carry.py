import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import spin_oracle as O
from paper_1811_00901_b200 import spin
rng = np.random.default_rng(21)
n = 4000
P = (rng.normal(size=(n, 3)) * 1e-3).astype(np.float32)
Nn = np.tile(np.array([0, 0, 1], np.float32), (n, 1))
cen = np.arange(0, n, 400, dtype=np.int32)
eng = spin.SpinEngine(torch.from_numpy(P).cuda(), torch.from_numpy(Nn).cuda())
for W, b in ((4, 1.0), (6, 0.0013), (6, 0.01), (8, 0.0013)):
    for mode in ("nearest", "bilinear"):
        g, st = eng.generate(torch.from_numpy(cen).cuda(), W, b, 0.5, mode=mode, stats=True)
        g = g.cpu().numpy().astype(np.float64)
        o = O.generate(P, Nn, cen, W, b, 0.5, O.NEAREST if mode == "nearest" else O.BILINEAR)
        err = np.abs(g - o).sum(axis=(1, 2)) / np.maximum(np.abs(o).sum(axis=(1, 2)), 1e-30)
        print(W, b, mode, "max rel", err.max(), "gpu sum", g[0].sum(), "ora sum", o[0].sum(), st["pairs_candidate"], st["pairs_accepted"], st["fp64_fallbacks"])
        if err.max() > 1e-5:
            print(np.round(g[0], 3)); print(np.round(o[0], 3))
